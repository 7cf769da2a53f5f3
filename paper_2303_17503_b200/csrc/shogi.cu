// Shogi batched step for sm_100a (no reference engine: PAPER.md:1278-1354 +
// DESIGN.md §3.4 conventions; CPU twin oracle/orc_shogi.c, perft-pinned).
//
// One warp per board. After lane 0 applies the action, the board is copied
// into shared memory in the MOVER'S FRAME with owner-relative colours (own
// pieces move "up"), so every rule below is side-agnostic:
//   * attack gather: for each target square, walk the 8 rays and the 4 knight
//     squares once and record (for both owners) the 14-bit mask of attacking
//     piece types and the attacker count -> the observation's attack planes,
//     the in-check plane and the checkers;
//   * legal moves: rays out of the own king give checkers, block squares and
//     pins; lanes own squares and emit step / slide / knight moves (promotion
//     choices, dead-piece rule), king moves against a king-transparent attack
//     test, and drops (nifu, dead squares, check blocks); a pawn drop in front
//     of the enemy king runs a warp-parallel mate test (uchifuzume);
//   * four-fold repetition through 64-bit position keys (scan of the ply log);
//   * observation: a 9639-bit stream (one bit per float, every plane is
//     binary) emitted as float4 through a LUT into the flat [n, 9, 9, 119]
//     stream (records are not 16-B aligned, edges use scalar stores).
#include "common.cuh"
#include "../../include/bbk.h"

namespace shogi {
#ifndef BBK_SHOGI_OBS_UNROLL
#define BBK_SHOGI_OBS_UNROLL 1   // r02: 1 = +2.7 % over 2, 4 = -1.8 %
#endif
constexpr int kShogiObsUnroll = BBK_SHOGI_OBS_UNROLL;   // observation chunk loop unroll (tuning knob)
using namespace bbk;

constexpr int A = 2187;
constexpr int NF = 81 * 119;        // 9639 floats per record
constexpr int kWarps = 4;
constexpr int BOARD_STRIDE = 96;
constexpr int MISC = 16;            // hand[2][7], stm, rep
constexpr int BLOOM_U64 = 32;       // 2048-bit repetition Bloom filter after each env's key log

enum { EMP = 0, FU = 1, KY, KE, GI, KI, KA, HI, OU, TO, NY, NK, NG, UM, RY };

// direction index d: 0 UP(-1,0) 1 UP_LEFT(-1,-1) 2 UP_RIGHT(-1,+1) 3 LEFT(0,-1)
// 4 RIGHT(0,+1) 5 DOWN(+1,0) 6 DOWN_LEFT(+1,-1) 7 DOWN_RIGHT(+1,+1)
__device__ __constant__ int8_t DR[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
__device__ __constant__ int8_t DC[8] = {0, -1, 1, -1, 1, 0, -1, 1};
__device__ __constant__ int8_t OPPD[8] = {5, 7, 6, 4, 3, 0, 2, 1};
// per type (index = type): step directions and slide directions (owner frame)
constexpr uint8_t STEP_T[16] = {0, 0x01, 0x00, 0x00, 0xC7, 0x3F, 0x00, 0x00, 0xFF, 0x3F, 0x3F, 0x3F, 0x3F, 0x39, 0xC6, 0};
constexpr uint8_t SLIDE_T[16] = {0, 0x00, 0x01, 0x00, 0x00, 0x00, 0xC6, 0x39, 0x00, 0, 0, 0, 0, 0xC6, 0x39, 0};
// ... packed 8 types per 64-bit word: a per-lane (divergent) type then indexes registers instead of
// the constant cache, which serialises distinct addresses (the attack gather reads it 8x per square)
constexpr uint64_t pack8(const uint8_t* t) {
    uint64_t v = 0;
    for (int i = 7; i >= 0; i--) v = (v << 8) | t[i];
    return v;
}
constexpr uint64_t STEP_LO = pack8(STEP_T), STEP_HI = pack8(STEP_T + 8);
constexpr uint64_t SLIDE_LO = pack8(SLIDE_T), SLIDE_HI = pack8(SLIDE_T + 8);
static_assert(STEP_LO == 0x00003FC700000100ull && SLIDE_HI == 0x0039C60000000000ull, "type table packing");
__device__ __forceinline__ uint32_t stepm(int ty) {
    return (uint32_t)(((ty & 8) ? STEP_HI : STEP_LO) >> ((ty & 7) * 8)) & 0xFFu;
}
__device__ __forceinline__ uint32_t slidem(int ty) {
    return (uint32_t)(((ty & 8) ? SLIDE_HI : SLIDE_LO) >> ((ty & 7) * 8)) & 0xFFu;
}
__device__ __constant__ uint8_t HAND_TYPE[7] = {FU, KY, KE, GI, KI, KA, HI};
__device__ __constant__ uint8_t HCAP[7] = {8, 4, 4, 4, 4, 2, 2};
__device__ __constant__ uint8_t HOFF[7] = {0, 8, 12, 16, 20, 24, 26};

struct WarpSmem {
    alignas(16) uint8_t mask[A + 48];
    alignas(16) uint32_t bits[NF / 32 + 4];
    uint8_t bd[96];            // mover frame, owner-relative: (owner << 4) | type, owner 0 = side to move
    uint8_t abs_[96];          // absolute board (state)
    uint16_t atk[2][81];       // attacking piece-type masks per owner
    uint8_t acnt[2][81];
    // occupancy of every line: rows 0-8 (bit = column), columns 9-17 (bit = row),
    // diagonals r - c = k - 8 at 18 + k and anti-diagonals r + c = k at 35 + k (bit = row)
    uint16_t line[52];
    uint8_t kesc[8];           // own king: neighbour d is a legal king destination
    uint64_t pinray[8][2];     // 81-bit ray masks (lo 64 | hi 17)
    int8_t pinsq[8];
    int8_t pinidx[96];         // square -> index of the king ray that pins the piece on it, or -1
    uint16_t task[320];        // own-piece move tasks: square | direction << 7 (8, 9 = knight jumps)
    uint8_t hand[16];          // hands [2][7] (absolute owners)
    // next-board prefetch (cp.async): board, misc, repetition Bloom filter
    alignas(16) uint8_t pf_abs[96];
    alignas(16) uint8_t pf_misc[16];
    alignas(16) uint32_t pf_bloom[2 * BLOOM_U64];
};

struct Params {
    bbk_cols in, out;
    bbk_shogi_state in_s, out_s;
    const int64_t* actions;
    const uint64_t* slot_keys;
    int64_t n, slot0;
    uint64_t key;
    int32_t max_steps;
    int force_reset;
    const uint8_t* load_board;   // kLoad: positions to start from, [n, 96] absolute codes / [n, 16] hands + stm
    const uint8_t* load_misc;
    int64_t tail_ctas;   // one-pass CTAs at the end of the grid (common.cuh pass_map)
};

struct M81 {   // 81-bit square set
    uint64_t lo, hi;
    __device__ __forceinline__ bool has(int s) const { return s < 64 ? (lo >> s) & 1ull : (hi >> (s - 64)) & 1ull; }
    __device__ __forceinline__ void set(int s) { if (s < 64) lo |= 1ull << s; else hi |= 1ull << (s - 64); }
};

__device__ __forceinline__ bool son(int r, int c) { return (unsigned)r < 9u && (unsigned)c < 9u; }
__device__ __forceinline__ int owner(uint8_t pc) { return pc >> 4; }
__device__ __forceinline__ int ptype(uint8_t pc) { return pc & 15; }
__device__ __forceinline__ bool promotable(int t) { return t == FU || t == KY || t == KE || t == GI || t == KA || t == HI; }
__device__ __forceinline__ int promote(int t) { return t <= GI ? t + 8 : t == KA ? UM : RY; }
__device__ __forceinline__ int unpromote(int t) { return (t >= TO && t <= NG) ? t - 8 : t == UM ? KA : t == RY ? HI : t; }

// Board accessor with up to three overridden squares (scratch positions).
struct Acc {
    const uint8_t* bd;
    int s0, s1, s2;
    uint8_t v0, v1, v2;
    __device__ __forceinline__ uint8_t operator()(int s) const {
        return s == s0 ? v0 : s == s1 ? v1 : s == s2 ? v2 : bd[s];
    }
};

// Does side w (0 = mover, 1 = opponent; owner-relative codes) attack square t?
__device__ bool attacked(const Acc& at, int t, int w) {
    const int r = t / 9, c = t - 9 * (t / 9);
    for (int d = 0; d < 8; d++) {
        int rr = r + DR[d], cc = c + DC[d], k = 1;
        while (son(rr, cc)) {
            uint8_t pc = at(rr * 9 + cc);
            if (pc) {
                if (owner(pc) == w) {
                    const int ty = ptype(pc), bit = w == 0 ? OPPD[d] : d;
                    if (((k == 1 ? (stepm(ty) | slidem(ty)) : slidem(ty)) >> bit) & 1) return true;
                }
                break;
            }
            rr += DR[d]; cc += DC[d]; k++;
        }
    }
    const int kr = w == 0 ? r + 2 : r - 2;   // knights: own move (-2, +-1), opponent (+2, +-1)
    for (int dc = -1; dc <= 1; dc += 2)
        if (son(kr, c + dc)) { uint8_t pc = at(kr * 9 + c + dc); if (pc && owner(pc) == w && ptype(pc) == KE) return true; }
    return false;
}

__device__ __forceinline__ int action_code(int dir, bool promo, int to) { return (dir + (promo ? 10 : 0)) * 81 + to; }

// ---------------------------------------------------------------- apply
// Apply the action (mover frame of `stm`) to the absolute board + hands. Lane 0.
__device__ void apply_action(uint8_t* abs_, uint8_t* hand /* [2][7] */, int stm, int a) {
    const int dir = a / 81, to = a - 81 * dir;
    auto fr = [&](int s) { return stm ? 80 - s : s; };
    const int tabs = fr(to);
    if (dir >= 20) {
        const int hi = dir - 20;
        hand[stm * 7 + hi] -= 1;
        abs_[tabs] = (uint8_t)((stm << 4) | HAND_TYPE[hi]);
        return;
    }
    const bool promo = dir >= 10;
    const int d = dir % 10;
    const int tr = to / 9, tc = to - 9 * (to / 9);
    int from;
    if (d >= 8) {
        from = (tr + 2) * 9 + tc + (d == 8 ? 1 : -1);   // knight came from (+2, -+1)
    } else {
        int rr = tr - DR[d], cc = tc - DC[d];
        from = rr * 9 + cc;
        while (!abs_[fr(from)]) { rr -= DR[d]; cc -= DC[d]; from = rr * 9 + cc; }
    }
    const int fabs = fr(from);
    const uint8_t pc = abs_[fabs], cap = abs_[tabs];
    if (cap) {
        int ct = unpromote(cap & 15);
        hand[stm * 7 + ct - 1] += 1;
    }
    abs_[tabs] = promo ? (uint8_t)((stm << 4) | promote(pc & 15)) : pc;
    abs_[fabs] = EMP;
}

__device__ __forceinline__ uint64_t sq_key(uint8_t pc, int s) {
    return mix64(0x5306100000000000ULL + (uint64_t)pc * 128 + (uint64_t)s);
}

// Occupancy bit masks of the 52 lines of the board. The squares are listed in four orders (rows,
// columns, diagonals r - c = k - 8, anti-diagonals r + c = k; each line contiguous, its squares by
// increasing row within a diagonal); three ballots per order give the occupancy as a 96-bit stream
// in that order, and lane j cuts line j out of its stream with one funnel shift (instead of nine
// byte loads and index arithmetic per line).
struct LineOrder {
    uint8_t sq[4][96];      // square at position o of order q (o >= 81: padding)
    uint8_t start[52], len[52], r0[52];   // line j: stream offset, length, row of its first bit
};
constexpr LineOrder make_line_order() {
    LineOrder t{};
    int o = 0;
    for (int r = 0; r < 9; r++)
        for (int c = 0; c < 9; c++) t.sq[0][o++] = (uint8_t)(r * 9 + c);
    o = 0;
    for (int c = 0; c < 9; c++)
        for (int r = 0; r < 9; r++) t.sq[1][o++] = (uint8_t)(r * 9 + c);
    for (int j = 0; j < 18; j++) { t.start[j] = (uint8_t)(9 * (j % 9)); t.len[j] = 9; t.r0[j] = 0; }
    for (int q = 2; q < 4; q++) {
        o = 0;
        for (int k = 0; k < 17; k++) {
            const int lo = k - 8 > 0 ? k - 8 : 0, hi = k < 8 ? k : 8;
            const int j = (q == 2 ? 18 : 35) + k;
            t.start[j] = (uint8_t)o; t.len[j] = (uint8_t)(hi - lo + 1); t.r0[j] = (uint8_t)lo;
            for (int r = lo; r <= hi; r++) t.sq[q][o++] = (uint8_t)(r * 9 + (q == 2 ? r - k + 8 : k - r));
        }
    }
    return t;
}
__device__ const LineOrder g_lines = make_line_order();

__device__ void build_lines(WarpSmem& S, int lane) {
    uint32_t w[4][3];
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
        for (int k = 0; k < 3; k++) {
            const int o = lane + 32 * k;
            const bool occ = o < 81 && S.bd[__ldg(&g_lines.sq[q][o])] != 0;
            w[q][k] = __ballot_sync(BBK_FULL, occ);
        }
    for (int j = lane; j < 52; j += 32) {
        const int q = j < 9 ? 0 : j < 18 ? 1 : j < 35 ? 2 : 3;
        const int st = __ldg(&g_lines.start[j]), ln = __ldg(&g_lines.len[j]), r0 = __ldg(&g_lines.r0[j]);
        const int wi = st >> 5;
        // select the order's words without a dynamically indexed register array
        const uint32_t a0 = q == 0 ? w[0][0] : q == 1 ? w[1][0] : q == 2 ? w[2][0] : w[3][0];
        const uint32_t a1 = q == 0 ? w[0][1] : q == 1 ? w[1][1] : q == 2 ? w[2][1] : w[3][1];
        const uint32_t a2 = q == 0 ? w[0][2] : q == 1 ? w[1][2] : q == 2 ? w[2][2] : w[3][2];
        const uint32_t lo = wi == 0 ? a0 : wi == 1 ? a1 : a2, hi = wi == 0 ? a1 : wi == 1 ? a2 : 0u;
        const uint32_t m = __funnelshift_r(lo, hi, st & 31) & ((1u << ln) - 1u);
        S.line[j] = (uint16_t)(m << r0);
    }
}

// Attack gather: for every target square, the piece types (14-bit mask) and
// number of pieces of each owner attacking it (obs planes 14-30 / 45-61). The
// first piece along each of the 8 rays comes from the line occupancy masks
// (highest set bit below / lowest above the target's position), so there are
// no data-dependent ray walks.
__device__ void gather_attacks(WarpSmem& S, int lane) {
    const uint8_t* bd = S.bd;
    for (int t = lane; t < 81; t += 32) {
        const int r = t / 9, c = t - 9 * r;
        uint32_t m0 = 0u, m1 = 0u, n0 = 0u, n1 = 0u;
        const uint32_t Lrow = S.line[r], Lcol = S.line[9 + c], Ldia = S.line[18 + r - c + 8], Lant = S.line[35 + r + c];
#pragma unroll
        for (int d = 0; d < 8; d++) {
            // line, position on it, and search side for direction d (DR/DC order)
            const uint32_t L = d == 0 || d == 5 ? Lcol : d == 3 || d == 4 ? Lrow : d == 1 || d == 7 ? Ldia : Lant;
            const int pos = d == 3 || d == 4 ? c : r;
            const bool lower = d <= 3;   // UP, UP_LEFT, UP_RIGHT, LEFT: towards lower indices
            const uint32_t m = lower ? L & ((1u << pos) - 1u) : L & ~((2u << pos) - 1u);
            if (!m) continue;
            const int bpos = lower ? 31 - __clz(m) : __ffs(m) - 1;
            const int q = d == 3 || d == 4 ? r * 9 + bpos
                        : d == 0 || d == 5 ? bpos * 9 + c
                        : d == 1 || d == 7 ? bpos * 9 + (bpos - r + c)
                                           : bpos * 9 + (r + c - bpos);
            const bool adj = lower ? bpos == pos - 1 : bpos == pos + 1;
            const uint8_t pc = bd[q];
            const int w = owner(pc), ty = ptype(pc), bit = w == 0 ? OPPD[d] : d;
            // branch-free update (the owner / hit pattern differs lane to lane)
            const uint32_t hit = ((adj ? (stepm(ty) | slidem(ty)) : slidem(ty)) >> bit) & 1u;
            const uint32_t tb = hit << ((ty - 1) & 15), h0 = hit & (uint32_t)(w == 0), h1 = hit & (uint32_t)(w != 0);
            m0 |= w == 0 ? tb : 0u; m1 |= w != 0 ? tb : 0u;
            n0 += h0; n1 += h1;
        }
        for (int dc = -1; dc <= 1; dc += 2) {
            if (son(r + 2, c + dc) && bd[(r + 2) * 9 + c + dc] == KE) { m0 |= 1u << (KE - 1); n0++; }
            if (son(r - 2, c + dc) && bd[(r - 2) * 9 + c + dc] == (16 | KE)) { m1 |= 1u << (KE - 1); n1++; }
        }
        S.atk[0][t] = (uint16_t)m0; S.atk[1][t] = (uint16_t)m1; S.acnt[0][t] = (uint8_t)n0; S.acnt[1][t] = (uint8_t)n1;
    }
}

// Observation: 9639-bit stream (bit f = float f of the record) then float4 emission.
__device__ void build_and_emit_obs(WarpSmem& S, const float4* lut, const uint8_t* hand, int side, bool in_check,
                                   float* obs_stream, int64_t b, int lane) {
    const uint8_t* bd = S.bd;
    // ---- observation bitstream
    for (int i = lane; i < NF / 32 + 4; i += 32) S.bits[i] = 0u;
    __syncwarp();
    // constant planes 62..118 (hand thresholds, check) as a 64-bit word at bit 62:
    // hand type hi of player `who` sets min(count, cap) ones at 28*who + HOFF[hi]
    uint64_t hp = 0ull;
#pragma unroll
    for (int who = 0; who < 2; who++) {
        const int own_side = who == 0 ? side : 1 - side;
#pragma unroll
        for (int hi = 0; hi < 7; hi++) {
            const uint32_t c = hand[own_side * 7 + hi], cap = HCAP[hi];
            const uint32_t n = c < cap ? c : cap;
            hp |= (uint64_t)((1u << n) - 1u) << (28 * who + HOFF[hi]);
        }
    }
    if (in_check) hp |= 1ull << (118 - 62);
    for (int pass = 0; pass < 4; pass++) {
        const int s = pass < 2 ? 2 * lane + pass : 64 + 2 * lane + (pass - 2);
        if (s < 81) {
            // 119-bit pattern of square s in two registers: piece (bit 31 owner + type - 1),
            // attacker types at 14 / 45, attacker-count thresholds at 28-30 / 59-61, then
            // the constant planes 62..118
            uint64_t plo = hp << 62, phi = hp >> 2;
            const uint8_t pc = bd[s];
            if (pc) {
                const int bit = 31 * owner(pc) + ptype(pc) - 1;   // < 62
                plo |= 1ull << bit;
            }
#pragma unroll
            for (int who = 0; who < 2; who++) {
                const int base = 31 * who + 14;
                const uint32_t n = S.acnt[who][s];
                const uint64_t thr = (n > 0 ? 1ull : 0ull) | (n > 1 ? 2ull : 0ull) | (n > 2 ? 4ull : 0ull);
                plo |= ((uint64_t)S.atk[who][s] << base) | (thr << (base + 14));
            }
            const uint32_t w[4] = {(uint32_t)plo, (uint32_t)(plo >> 32), (uint32_t)phi, (uint32_t)(phi >> 32)};
            const int off = 119 * s, wi = off >> 5, sh = off & 31;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                S.bits[wi + j] |= w[j] << sh;
                if (sh) S.bits[wi + j + 1] |= w[j] >> (32 - sh);
            }
        }
        __syncwarp();
    }
#ifndef BBK_SHOGI_OBS_V8
#define BBK_SHOGI_OBS_V8 1
#endif
    if (obs_stream && BBK_SHOGI_OBS_V8) {   // 32-byte stores over the 32-B aligned interior
        const int64_t F0 = b * (int64_t)NF;
        const int head = (int)((8 - (F0 & 7)) & 7);
        const int nchunk = (NF - head) >> 3;
        const int tail0 = head + 8 * nchunk;
        float* rec = obs_stream + F0;
        if (lane < head || (lane >= 8 && lane - 8 < NF - tail0)) {   // at most 7 edge floats each side
            const uint32_t fi = lane < 8 ? (uint32_t)lane : (uint32_t)(tail0 + lane - 8);
            rec[fi] = (float)((S.bits[fi >> 5] >> (fi & 31)) & 1u);
        }
        // chunk j = lane + 32 m starts at bit head + 8 lane + 256 m: lane-constant shift
        float* o8 = rec + head;
        const uint32_t q0 = (uint32_t)(head + 8 * lane), sh = q0 & 31u;
        const uint32_t* wp = S.bits + (q0 >> 5);
#pragma unroll kShogiObsUnroll
        for (int j = lane; j < nchunk; j += 32, wp += 8) {
            const uint32_t t = __funnelshift_r(wp[0], wp[1], sh);
            const float4 lo = lut[t & 15u], hi = lut[(t >> 4) & 15u];
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o8 + 8 * j), "f"(lo.x), "f"(lo.y),
                         "f"(lo.z), "f"(lo.w), "f"(hi.x), "f"(hi.y), "f"(hi.z), "f"(hi.w) : "memory");
        }
    } else if (obs_stream) {   // flat [n, 9, 9, 119] stream; records are not 16-B aligned
        const int64_t F0 = b * (int64_t)NF;
        const int head = (int)((4 - (F0 & 3)) & 3);
        const int nchunk = (NF - head) >> 2;
        const int tail0 = head + 4 * nchunk;
        float* rec = obs_stream + F0;
        if (lane < head || (lane >= 4 && lane - 4 < NF - tail0)) {
            const uint32_t fi = lane < 4 ? (uint32_t)lane : (uint32_t)(tail0 + lane - 4);
            rec[fi] = (float)((S.bits[fi >> 5] >> (fi & 31)) & 1u);
        }
        // chunk j = lane + 32 m starts at bit head + 4 lane + 128 m: lane-constant shift
        float4* o4 = reinterpret_cast<float4*>(rec + head);
        const uint32_t q0 = (uint32_t)(head + 4 * lane), sh = q0 & 31u;
        const uint32_t* wp = S.bits + (q0 >> 5);
#pragma unroll 4
        for (int j = lane; j < nchunk; j += 32, wp += 4) o4[j] = lut[__funnelshift_r(wp[0], wp[1], sh) & 15u];
    }
}

// One scalar field of board b per lane (lanes 0-3), loaded a board ahead.
__device__ __forceinline__ FieldRef field_ref(const Params& p, int lane) {
    switch (lane) {
        case 0: return field_of(p.in.terminated, 0u);
        case 1: return field_of(p.in.player_to_role, 1u);
        case 2: return field_of(p.in.step_count, 2u);
        case 3: return field_of(p.actions, 3u);
        case 4: return field_of(p.in.truncated, 0u);
        default: return no_field();
    }
}

// cp.async board b's board, misc and repetition Bloom filter into the prefetch area.
__device__ __forceinline__ void issue_prefetch(WarpSmem& S, const Params& p, int64_t b, int lane) {
    const char* src = nullptr;
    uint32_t dst = 0u;
    if (lane < 6) {
        src = reinterpret_cast<const char*>(p.in_s.board + b * BOARD_STRIDE) + 16 * lane;
        dst = (uint32_t)__cvta_generic_to_shared(S.pf_abs) + 16u * lane;
    } else if (lane == 6) {
        src = reinterpret_cast<const char*>(p.in_s.misc + b * MISC);
        dst = (uint32_t)__cvta_generic_to_shared(S.pf_misc);
    } else if (lane < 7 + 16) {
        const uint64_t* hist = p.out_s.hist + b * (int64_t)p.out_s.hist_cap;
        src = reinterpret_cast<const char*>(hist + p.out_s.hist_cap - BLOOM_U64) + 16 * (lane - 7);
        dst = (uint32_t)__cvta_generic_to_shared(S.pf_bloom) + 16u * (lane - 7);
    }
    if (src) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    asm volatile("cp.async.commit_group;");
}

// kLoad: a reset that starts from p.load_board / p.load_misc instead of the initial position
// (bbk_shogi_load, the device twin of the oracle's orc_shogi_set_sfen test hook); a separate
// instantiation so the hot kernel's code is unchanged.
template <bool kLoad>
#ifndef BBK_SHOGI_MIN_CTAS
#define BBK_SHOGI_MIN_CTAS 9   // r02 (after the grid / line / unroll changes): 9 = +1.7 % over 8 (56 registers), 10: -6 %
#endif
__global__ void __launch_bounds__(kWarps * 32, BBK_SHOGI_MIN_CTAS) step_kernel(Params p) {
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
    const int cap = p.out_s.hist_cap;
    unsigned long long eps = 0;
    uint8_t* hand = S.hand;
    const int64_t b0 = pm.b0;
    uint64_t cur = 0ull;   // this board's scalar fields (lane j holds field j)
    bool pf_ready = false;
    const FieldRef fref = field_ref(p, lane_id());
    for (int64_t b = b0; b < bend; b += nwarps) {
        if (!p.force_reset && !pf_ready) {   // first board of the warp: fetch synchronously
            cur = load_field(fref, b);
            issue_prefetch(S, p, b, lane);
        }
        const int64_t nb = b + nwarps;   // the next board's scalars are in flight meanwhile
        const uint64_t nxt = (!p.force_reset && nb < bend) ? load_field(fref, nb) : 0ull;
        const uint32_t f_term = __shfl_sync(BBK_FULL, (uint32_t)cur, 0) | (__shfl_sync(BBK_FULL, (uint32_t)cur, 4) << 8);
        const bool reset = p.force_reset || (f_term & 0xFFFFu) != 0u;
        if (!p.force_reset) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        const uint64_t k = slot_key(p.slot_keys, p.key, p.slot0, b);
        uint64_t* hist = p.out_s.hist + b * (int64_t)cap;
        int8_t p2r0, p2r1;
        int stm, step;
        if (reset) {
            int c = (int)(child(k, 0) % 2ull);
            p2r0 = (int8_t)c; p2r1 = (int8_t)(1 - c);
            // lnsgkgsnl/1r5b1/ppppppppp/9/9/9/PPPPPPPPP/1B5R1/LNSGKGSNL (White = owner 1 at the top)
            if (kLoad) {
                for (int s = lane; s < 96; s += 32) S.abs_[s] = s < 81 ? p.load_board[b * 96 + s] : (uint8_t)0;
                if (lane < 16) hand[lane] = lane < 14 ? p.load_misc[b * 16 + lane] : (uint8_t)0;
                stm = p.load_misc[b * 16 + 14] & 1;
            } else {
                constexpr uint64_t back = 0x234585432ull;   // KY KE GI KI OU KI GI KE KY, nibble c = file c
                for (int s = lane; s < 96; s += 32) {
                    uint8_t v = 0;
                    if (s < 81) {
                        int r = s / 9, cc = s - 9 * r;
                        const uint8_t bk = (uint8_t)((back >> (4 * cc)) & 15u);
                        if (r == 0) v = (uint8_t)(16 | bk);
                        else if (r == 1) v = cc == 1 ? (uint8_t)(16 | HI) : cc == 7 ? (uint8_t)(16 | KA) : 0;
                        else if (r == 2) v = 16 | FU;
                        else if (r == 6) v = FU;
                        else if (r == 7) v = cc == 1 ? KA : cc == 7 ? HI : 0;
                        else if (r == 8) v = bk;
                    }
                    S.abs_[s] = v;
                }
                if (lane < 16) hand[lane] = 0;
                stm = 0;
            }
            step = 0;
            __syncwarp();
        } else {
            const uint32_t f_p2r = __shfl_sync(BBK_FULL, (uint32_t)cur, 1);
            const int f_step = (int)__shfl_sync(BBK_FULL, (uint32_t)cur, 2);
            const int f_act = (int)shfl64(cur, 3);
            p2r0 = (int8_t)(f_p2r & 0xFF); p2r1 = (int8_t)(f_p2r >> 8);
            for (int s = lane; s < 96; s += 32) S.abs_[s] = S.pf_abs[s];
            if (lane < 16) hand[lane] = S.pf_misc[lane];
            stm = S.pf_misc[14];
            step = f_step + 1;
            __syncwarp();
            if (lane == 0) apply_action(S.abs_, hand, stm, f_act);
            stm ^= 1;
            __syncwarp();
        }
        const int side = stm;
        // mover-frame, owner-relative board
        for (int s = lane; s < 81; s += 32) {
            uint8_t v = S.abs_[side ? 80 - s : s];
            S.bd[s] = v ? (uint8_t)((((v >> 4) ^ side) << 4) | (v & 15)) : (uint8_t)0;
        }
        for (int i = lane; i < (A + 48) / 16; i += 32) reinterpret_cast<uint4*>(S.mask)[i] = make_uint4(0, 0, 0, 0);
        for (int i = lane; i < 96 / 4; i += 32) reinterpret_cast<uint32_t*>(S.pinidx)[i] = 0xFFFFFFFFu;
        __syncwarp();
        const uint8_t* bd = S.bd;
        const int64_t mstart = b * (int64_t)A;
        uint8_t* mk = S.mask + (mstart & 15);   // mask byte i staged at the destination's 16-byte phase
        // ---- king squares, attack gather (both owners), pawn columns
        int ksq = -1, oksq = -1;
        uint32_t pawncols = 0u;
        for (int s = lane; s < 81; s += 32) {
            uint8_t pc = bd[s];
            if (pc == OU) ksq = s;
            if (pc == (16 | OU)) oksq = s;
            if (pc == FU) pawncols |= 1u << (s % 9);
        }
        {
            unsigned bk = __ballot_sync(BBK_FULL, ksq >= 0), bo = __ballot_sync(BBK_FULL, oksq >= 0);
            ksq = __shfl_sync(BBK_FULL, ksq, bk ? __ffs(bk) - 1 : 0);
            oksq = __shfl_sync(BBK_FULL, oksq, bo ? __ffs(bo) - 1 : 0);
            pawncols = __reduce_or_sync(BBK_FULL, pawncols);
        }
        build_lines(S, lane);
        __syncwarp();
        gather_attacks(S, lane);
        __syncwarp();
        const bool in_check = ksq >= 0 && S.acnt[1][ksq] > 0;
        // ---- checkers / block squares / pins along the 8 rays out of the king
        bool checker = false;
        M81 block{0ull, 0ull};
        const int kr = ksq / 9, kc = ksq - 9 * (ksq / 9);
        if (lane < 8) {
            const int d = lane;
            int rr = kr + DR[d], cc = kc + DC[d], kk = 1, own = -1;
            M81 ray{0ull, 0ull};
            int8_t pin = -1;
            M81 pray{0ull, 0ull};
            while (son(rr, cc)) {
                const int s = rr * 9 + cc;
                ray.set(s);
                const uint8_t pc = bd[s];
                if (pc) {
                    const int ty = ptype(pc);
                    if (own < 0) {
                        if (owner(pc) == 0) own = s;
                        else {
                            if (((kk == 1 ? (stepm(ty) | slidem(ty)) : slidem(ty)) >> d) & 1) { checker = true; block = ray; }
                            break;
                        }
                    } else {
                        if (owner(pc) == 1 && ((slidem(ty) >> d) & 1)) { pin = (int8_t)own; pray = ray; }
                        break;
                    }
                }
                rr += DR[d]; cc += DC[d]; kk++;
            }
            S.pinsq[d] = pin;
            if (pin >= 0) S.pinidx[pin] = (int8_t)d;
            S.pinray[d][0] = pray.lo; S.pinray[d][1] = pray.hi;
            // king destination d: on board, not own, not attacked with the king lifted
            const int tr = kr + DR[d], tc = kc + DC[d];
            bool ok = false;
            if (son(tr, tc)) {
                const int t = tr * 9 + tc;
                const uint8_t q = bd[t];
                if (!(q && owner(q) == 0) && S.acnt[1][t] == 0) {
                    // the gather saw every attacker except a slider x-raying through our king:
                    // walk once from the king away from t
                    const int od = OPPD[d];
                    int xr = kr + DR[od], xc = kc + DC[od];
                    ok = true;
                    while (son(xr, xc)) {
                        const uint8_t pc = bd[xr * 9 + xc];
                        if (pc) { ok = !(owner(pc) == 1 && ((slidem(ptype(pc)) >> od) & 1)); break; }
                        xr += DR[od]; xc += DC[od];
                    }
                }
            }
            S.kesc[d] = ok;
        } else if (lane < 10) {   // knight checkers: opponent knights at (kr-2, kc-+1)
            const int cc = kc + (lane == 8 ? -1 : 1), rr = kr - 2;
            if (son(rr, cc) && bd[rr * 9 + cc] == (16 | KE)) { checker = true; block.set(rr * 9 + cc); }
        }
        const int nchecks = __popc(__ballot_sync(BBK_FULL, checker));
        M81 chk;
        chk.lo = ((uint64_t)__reduce_or_sync(BBK_FULL, (uint32_t)(block.lo >> 32)) << 32) |
                 __reduce_or_sync(BBK_FULL, (uint32_t)block.lo);
        chk.hi = __reduce_or_sync(BBK_FULL, (uint32_t)block.hi);
        if (nchecks == 0) { chk.lo = ~0ull; chk.hi = ~0ull; }
        else if (nchecks >= 2) { chk.lo = 0ull; chk.hi = 0ull; }
        __syncwarp();
        // ---- moves of own pieces: (piece, direction) tasks strided over the lanes, so the
        //      few pieces and their uneven rays do not serialise the warp
        int cnt = 0;
        if (lane < 8 && ksq >= 0 && S.kesc[lane]) {   // king destinations (lane = direction)
            mk[action_code(lane, false, ksq + DR[lane] * 9 + DC[lane])] = 1;
            cnt++;
        }
        {
            uint32_t dirs[3];
            int mine = 0;
#pragma unroll
            for (int j = 0; j < 3; j++) {
                const int sq = lane + 32 * j;
                const uint8_t pc = sq < 81 ? bd[sq] : (uint8_t)0;
                const int ty = ptype(pc);
                dirs[j] = (!pc || owner(pc) != 0 || ty == OU) ? 0u : ty == KE ? 0x300u : (uint32_t)(stepm(ty) | slidem(ty));
                mine += __popc(dirs[j]);
            }
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(BBK_FULL, incl, o);
                if (lane >= o) incl += t;
            }
            const int ntask = __shfl_sync(BBK_FULL, incl, 31);
            BBK_CHECK(ntask <= 320);   // task list capacity (WarpSmem::task)
            int k = incl - mine;
#pragma unroll
            for (int j = 0; j < 3; j++)
                for (uint32_t m = dirs[j]; m; m &= m - 1) S.task[k++] = (uint16_t)((lane + 32 * j) | ((__ffs(m) - 1) << 7));
            __syncwarp();
            for (int i = lane; i < ntask; i += 32) {
                const int tk = S.task[i], sq = tk & 127, d = tk >> 7;
                const int ty = ptype(bd[sq]), r = sq / 9, c = sq - 9 * (sq / 9);
                M81 allow = chk;
                const int pi = S.pinidx[sq];
                if (pi >= 0) { allow.lo &= S.pinray[pi][0]; allow.hi &= S.pinray[pi][1]; }
                auto emit = [&](int dd, int to) {
                    if (!allow.has(to)) return;
                    const int trow = to / 9;
                    const bool can_promo = promotable(ty) && (r <= 2 || trow <= 2);
                    const bool must = (ty == FU || ty == KY) ? trow == 0 : ty == KE ? trow <= 1 : false;
                    if (can_promo) { mk[action_code(dd, true, to)] = 1; cnt++; }
                    if (!must) { mk[action_code(dd, false, to)] = 1; cnt++; }
                };
                if (d >= 8) {   // knight jump (-2, -1) / (-2, +1)
                    const int rr = r - 2, cc = c + (d == 9 ? 1 : -1);
                    if (son(rr, cc)) {
                        const uint8_t q = bd[rr * 9 + cc];
                        if (!(q && owner(q) == 0)) emit(d, rr * 9 + cc);
                    }
                    continue;
                }
                const bool slide = (slidem(ty) >> d) & 1;
                int rr = r + DR[d], cc = c + DC[d];
                while (son(rr, cc)) {
                    const int to = rr * 9 + cc;
                    const uint8_t q = bd[to];
                    if (q && owner(q) == 0) break;
                    emit(d, to);
                    if (q || !slide) break;
                    rr += DR[d]; cc += DC[d];
                }
            }
        }
        // ---- drops (block squares only when in single check; none in double check)
        const M81 dropok = chk;   // the checker's own square is occupied, so drops only block
        const int my = side * 7;
        for (int s = lane; s < 81; s += 32) {
            if (bd[s]) continue;
            if (nchecks >= 2) continue;
            if (nchecks == 1 && !dropok.has(s)) continue;
            const int r = s / 9, c = s - 9 * r;
            for (int hi = 0; hi < 7; hi++) {
                if (!hand[my + hi]) continue;
                const int ty = HAND_TYPE[hi];
                if ((ty == FU || ty == KY) && r == 0) continue;
                if (ty == KE && r <= 1) continue;
                if (ty == FU) {
                    if ((pawncols >> c) & 1u) continue;
                    if (oksq >= 0 && s == oksq + 9) continue;   // uchifuzume candidate: decided below
                }
                mk[action_code(20 + hi, false, s)] = 1;
                cnt++;
            }
        }
        // uchifuzume: pawn drop on the square in front of the enemy king
        {
            const int D = oksq + 9;
            bool cand = oksq >= 0 && oksq + 9 < 81 && hand[my + 0] && !bd[D] && !((pawncols >> (D % 9)) & 1u) &&
                        nchecks < 2 && (nchecks == 0 || chk.has(D));
            if (cand) {
                // after the drop: can the enemy king escape, or can an enemy piece take the pawn?
                bool reply = false;
                const int okr = oksq / 9, okc = oksq - 9 * okr;
                if (lane < 8) {
                    const int tr = okr + DR[lane], tc = okc + DC[lane];
                    if (son(tr, tc)) {
                        const int t = tr * 9 + tc;
                        const uint8_t q = t == D ? (uint8_t)FU : bd[t];
                        if (!(q && owner(q) == 1)) {
                            Acc at{bd, D, oksq, t, (uint8_t)FU, 0, (uint8_t)(16 | OU)};
                            reply = !attacked(at, t, 0);
                        }
                    }
                } else if (lane < 18) {   // lanes 8..15: ray attackers of D; 16,17: knights
                    const int dr_ = D / 9, dc_ = D - 9 * (D / 9);
                    int from = -1;
                    if (lane < 16) {
                        const int d = lane - 8;
                        int rr = dr_ + DR[d], cc = dc_ + DC[d], kk = 1;
                        while (son(rr, cc)) {
                            const uint8_t pc = bd[rr * 9 + cc];
                            if (pc) {
                                const int ty = ptype(pc);
                                if (owner(pc) == 1 && ty != OU && (((kk == 1 ? (stepm(ty) | slidem(ty)) : slidem(ty)) >> d) & 1))
                                    from = rr * 9 + cc;
                                break;
                            }
                            rr += DR[d]; cc += DC[d]; kk++;
                        }
                    } else {
                        const int rr = dr_ - 2, cc = dc_ + (lane == 16 ? -1 : 1);
                        if (son(rr, cc) && bd[rr * 9 + cc] == (16 | KE)) from = rr * 9 + cc;
                    }
                    if (from >= 0) {
                        Acc at{bd, D, from, -1, bd[from], 0, 0};
                        reply = !attacked(at, oksq, 0);
                    }
                }
                const bool any_reply = __any_sync(BBK_FULL, reply);
                if (lane == 0 && any_reply) { mk[action_code(20, false, D)] = 1; cnt++; }
            }
        }
        const int nlegal = warp_sum(cnt);
        // ---- position key + four-fold repetition
        uint64_t key = 0ull;
        for (int s = lane; s < 81; s += 32) { uint8_t v = S.abs_[s]; if (v) key ^= sq_key(v, s); }
        if (lane < 14 && hand[lane]) {
            const int c = lane / 7, i = lane - 7 * c;
            key ^= mix64(0x5306200000000000ULL + (uint64_t)(c * 8 + i) * 32 + hand[lane]);
        }
        key = warp_xor64(key);
        if (side) key ^= mix64(0x5306300000000000ULL);
        // four-fold repetition: 2048-bit Bloom filter of the ply log (stored after it), exact
        // scan of the log only on a Bloom hit (identical answers to scanning every key)
        uint32_t* bloom = reinterpret_cast<uint32_t*>(hist + cap - BLOOM_U64);
        const uint32_t i1 = (uint32_t)key & 2047u, i2 = (uint32_t)(key >> 11) & 2047u;
        if (step == 0) {
            for (int j = lane; j < 2 * BLOOM_U64; j += 32) bloom[j] = 0u;
            __syncwarp();
        }
        int reps = 0;
        const uint32_t* pb = S.pf_bloom;   // prefetched copy of this env's filter
        if (step > 0 && ((pb[i1 >> 5] >> (i1 & 31)) & (pb[i2 >> 5] >> (i2 & 31)) & 1u)) {
            for (int j = lane; j < step; j += 32) reps += hist[j] == key;
            reps = warp_sum(reps);
        }
        __syncwarp();   // the prefetch area is free now: issue the next board's state
        pf_ready = false;
        if (!p.force_reset && nb < bend) {
            issue_prefetch(S, p, nb, lane);
            cur = nxt;
            pf_ready = true;
        }
        BBK_CHECK(step < cap - BLOOM_U64);   // the key log ends where its Bloom filter starts
        if (lane == 0) {
            hist[step] = key;
            atomicOr(&bloom[i1 >> 5], 1u << (i1 & 31));
            atomicOr(&bloom[i2 >> 5], 1u << (i2 & 31));
        }
        bool terminal = false;
        float rr0 = 0.0f, rr1 = 0.0f;
        if (nlegal == 0) {   // no legal move: the side to move loses
            terminal = true;
            if (side == 0) { rr0 = -1.0f; rr1 = 1.0f; } else { rr0 = 1.0f; rr1 = -1.0f; }
        } else if (reps >= 3) {
            terminal = true;
        }
        const bool truncated = !terminal && step >= p.max_steps;
        eps += (terminal || truncated) ? 1 : 0;
        if (p.out.next_actions) {   // fused agents.random_actions on the new mask (still in shared memory)
            const int64_t a = warp_sample_bytes<true>(mk, A, (terminal || truncated) ? 0 : nlegal, p.out.next_key,
                                                p.slot0 + b);
            if (lane == 0) p.out.next_actions[b] = a;
        }
        build_and_emit_obs(S, lut, hand, side, in_check, p.out.observation, b, lane);
        // ---- mask emission (flat byte stream; records are not 16-B aligned)
        __syncwarp();
        if (terminal || truncated)
            for (int i = lane; i < (A + 48) / 16; i += 32) reinterpret_cast<uint4*>(S.mask)[i] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        warp_emit_bytes(p.out.legal_action_mask, mstart, A, S.mask);
        // ---- state + columns
        uint8_t* ob = p.out_s.board + b * BOARD_STRIDE;
        for (int s = lane; s < 96; s += 32) ob[s] = S.abs_[s];
        if (lane < 14) p.out_s.misc[b * MISC + lane] = hand[lane];
        const int rep = reps > 3 ? 3 : reps;
        if (lane == 0) {
            uint8_t* m = p.out_s.misc + b * MISC;
            m[14] = (uint8_t)side; m[15] = (uint8_t)rep;
            float r0 = 0.0f, r1 = 0.0f;
            if (!truncated && (rr0 != 0.0f || rr1 != 0.0f)) { r0 = p2r0 == 0 ? rr0 : rr1; r1 = p2r1 == 0 ? rr0 : rr1; }
            p.out.rewards[2 * b] = r0; p.out.rewards[2 * b + 1] = r1;
            p.out.terminated[b] = terminal; p.out.truncated[b] = truncated;
            p.out.step_count[b] = step;
            p.out.current_player[b] = p2r0 == side ? 0 : 1;
            p.out.player_to_role[2 * b] = p2r0; p.out.player_to_role[2 * b + 1] = p2r1;
        }
        __syncwarp();
    }
    if (p.out.episodes && lane_id() == 0 && eps) atomicAdd(p.out.episodes, eps);
}

// observe(state, player) for an explicit role per slot (no history planes in shogi).
__global__ void __launch_bounds__(kWarps * 32) observe_kernel(bbk_shogi_state st, const uint8_t* role, float* obs,
                                                              int64_t n) {
    __shared__ WarpSmem sm[kWarps];
    __shared__ float4 lut[16];
    if (threadIdx.x < 16) {
        uint32_t q = threadIdx.x;
        lut[q] = make_float4((float)(q & 1), (float)((q >> 1) & 1), (float)((q >> 2) & 1), (float)((q >> 3) & 1));
    }
    __syncthreads();
    WarpSmem& S = sm[threadIdx.x >> 5];
    const int lane = lane_id();
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    for (int64_t b = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); b < n; b += nwarps) {
        const int side = role[b];
        const uint8_t* ib = st.board + b * BOARD_STRIDE;
        for (int s = lane; s < 81; s += 32) {
            uint8_t v = ib[side ? 80 - s : s];
            S.bd[s] = v ? (uint8_t)((((v >> 4) ^ side) << 4) | (v & 15)) : (uint8_t)0;
        }
        uint8_t hand[14];
        const uint8_t* m = st.misc + b * MISC;
#pragma unroll
        for (int j = 0; j < 14; j++) hand[j] = m[j];
        __syncwarp();
        build_lines(S, lane);
        __syncwarp();
        gather_attacks(S, lane);
        int ksq = -1;
        for (int s = lane; s < 81; s += 32) if (S.bd[s] == OU) ksq = s;
        unsigned bk = __ballot_sync(BBK_FULL, ksq >= 0);
        ksq = __shfl_sync(BBK_FULL, ksq, bk ? __ffs(bk) - 1 : 0);
        const bool in_check = bk && S.acnt[1][ksq] > 0;
        build_and_emit_obs(S, lut, hand, side, in_check, obs, b, lane);
        __syncwarp();
    }
}

#ifndef BBK_SHOGI_GRID_BOARDS
#define BBK_SHOGI_GRID_BOARDS 1   // boards per warp per launch (common.cuh step_grid); 0: persistent grid (r02: 1 = +2.3 %, 2 = +0.5 %, 4 = -2.6 %)
#endif
#ifndef BBK_SHOGI_TAIL_PCT
#define BBK_SHOGI_TAIL_PCT 0   // one-pass CTAs at the end of the grid, % of the resident CTAs
#endif
template <bool kLoad>
static void launch_grid(const Params& p, cudaStream_t s) {
    const int64_t need = (p.n + kWarps - 1) / kWarps;
    const int64_t resident = resident_ctas(step_kernel<kLoad>, kWarps * 32, 0);
    const int64_t grid = wave_grid(resident, need, BBK_SHOGI_GRID_BOARDS);
    Params q = p;
    q.tail_ctas = tail_ctas(grid, resident, BBK_SHOGI_TAIL_PCT);
    step_kernel<kLoad><<<(unsigned)grid, kWarps * 32, 0, s>>>(q);
}
static int launch(const Params& p, cudaStream_t s) {
    if (p.load_board) launch_grid<true>(p, s);
    else launch_grid<false>(p, s);
    return (int)cudaGetLastError();
}

}  // namespace shogi

extern "C" {

int bbk_shogi_init(const bbk_cols* out, const bbk_shogi_state* out_s, int64_t n, int64_t slot0, uint64_t key_state,
                   const uint64_t* slot_keys, int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    shogi::Params p{};
    p.out = *out; p.out_s = *out_s; p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.force_reset = 1;
    return shogi::launch(p, (cudaStream_t)stream);
}

int bbk_shogi_load(const bbk_cols* out, const bbk_shogi_state* out_s, const uint8_t* boards, const uint8_t* misc,
                   int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys, int32_t max_steps,
                   void* stream) {
    if (n <= 0) return 0;
    if (!boards || !misc) return (int)cudaErrorInvalidValue;
    shogi::Params p{};
    p.out = *out; p.out_s = *out_s; p.slot_keys = slot_keys; p.n = n; p.slot0 = slot0; p.key = key_state;
    p.max_steps = max_steps; p.force_reset = 1; p.load_board = boards; p.load_misc = misc;
    return shogi::launch(p, (cudaStream_t)stream);
}

int bbk_shogi_step(const bbk_cols* in, const bbk_shogi_state* in_s, const bbk_cols* out, const bbk_shogi_state* out_s,
                   const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                   int32_t max_steps, void* stream) {
    if (n <= 0) return 0;
    shogi::Params p{};
    p.in = *in; p.in_s = *in_s; p.out = *out; p.out_s = *out_s; p.actions = actions; p.slot_keys = slot_keys;
    p.n = n; p.slot0 = slot0; p.key = key_state; p.max_steps = max_steps; p.force_reset = 0;
    return shogi::launch(p, (cudaStream_t)stream);
}

int bbk_shogi_observe(const bbk_shogi_state* s, const int32_t* step_count, const uint8_t* role, float* obs, int64_t n,
                      void* stream) {
    (void)step_count;
    if (n <= 0) return 0;
    int64_t grid = (n + shogi::kWarps - 1) / shogi::kWarps;
    if (grid > 148 * 8) grid = 148 * 8;
    shogi::observe_kernel<<<(unsigned)grid, shogi::kWarps * 32, 0, (cudaStream_t)stream>>>(*s, role, obs, n);
    return (int)cudaGetLastError();
}

}  // extern "C"

// checked builds: this translation unit's failed-check word (common.cuh BBK_CHECK)
BBK_CHECK_READER(bbk_tu_fail_shogi)
