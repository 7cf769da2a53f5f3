// The reference's small engines as per-thread device state machines
// (SURVEY §8f rank 4): tic-tac-toe (games/tictactoe.py), Connect Four
// (connect_four.py), Othello (othello.py), Hex (hexgame.py), 2048
// (play2048.py), Kuhn poker (kuhn_poker.py) and Leduc hold'em
// (leduc_holdem.py). Each engine keeps its Core in a 48-byte per-slot blob
// and restates init_core / apply / mask / observe / encode of its reference
// module; the env-core logic around them (reset, truncation, rewards by
// player, mask zeroing, core.py:192-220, 353-386) lives in small.cu.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace small {
using namespace bbk;

constexpr int kStateBytes = 48;

struct Mask128 {
    uint64_t lo, hi;
    __device__ __forceinline__ bool has(int a) const { return a < 64 ? (lo >> a) & 1ull : (hi >> (a - 64)) & 1ull; }
    __device__ __forceinline__ int count() const { return __popcll(lo) + __popcll(hi); }
};

struct St {   // the 48-byte blob, accessed as bytes / 64-bit words
    union {
        uint8_t b[kStateBytes];
        uint64_t q[kStateBytes / 8];
    };
};

// Outcome of apply(): terminal flag and role rewards (Core.rewards).
struct Out {
    bool terminal;
    float r0, r1;
};

__device__ __forceinline__ Out win_for(int mover) { return Out{true, mover == 0 ? 1.0f : -1.0f, mover == 0 ? -1.0f : 1.0f}; }

// Lehmer decoding of RngKey.permutation(n) (rng.py:107-117): code = state % n!.
__device__ __forceinline__ void permutation(uint64_t state, int n, int* out) {
    uint64_t fact[8] = {1, 1, 2, 6, 24, 120, 720, 5040};
    uint64_t code = state % fact[n];
    int pool[8];
    for (int i = 0; i < n; i++) pool[i] = i;
    int m = n;
    for (int radix = n - 1, k = 0; radix >= 0; radix--, k++) {
        const int digit = (int)(code / fact[radix]);
        code %= fact[radix];
        out[k] = pool[digit];
        for (int j = digit; j < m - 1; j++) pool[j] = pool[j + 1];
        m--;
    }
}

// ------------------------------------------------------------ tic-tac-toe
// blob: board[9] (0 empty, 1 / 2 = role 0 / 1), role (9)   (tictactoe.py:21-62)
struct TicTacToe {
    static constexpr int A = 9, P = 2, OBS = 18;
    __device__ static int role(const St& s) { return s.b[9]; }
    __device__ static bool init(St& s, uint64_t) { for (int i = 0; i < 10; i++) s.b[i] = 0; return false; }
    __device__ static Out apply(St& s, int a, uint64_t) {
        const int mover = s.b[9], mark = mover + 1;
        s.b[a] = (uint8_t)mark;
        const uint8_t L[8][3] = {{0, 1, 2}, {3, 4, 5}, {6, 7, 8}, {0, 3, 6}, {1, 4, 7}, {2, 5, 8}, {0, 4, 8}, {2, 4, 6}};
        bool win = false, full = true;
        for (int l = 0; l < 8; l++)
            win |= s.b[L[l][0]] == mark && s.b[L[l][1]] == mark && s.b[L[l][2]] == mark;
        for (int i = 0; i < 9; i++) full &= s.b[i] != 0;
        s.b[9] = (uint8_t)(1 - mover);
        if (win) return win_for(mover);
        return Out{full, 0.0f, 0.0f};
    }
    __device__ static Mask128 mask(const St& s) {
        uint64_t m = 0;
        for (int i = 0; i < 9; i++) m |= (uint64_t)(s.b[i] == 0) << i;
        return Mask128{m, 0};
    }
    __device__ static void observe(const St& s, int role, bool, float* o) {   // (3, 3, 2)
        for (int i = 0; i < 9; i++) {
            o[2 * i] = s.b[i] == role + 1 ? 1.0f : 0.0f;
            o[2 * i + 1] = s.b[i] == 2 - role ? 1.0f : 0.0f;
        }
    }
    // float f of the observation record (for warp-cooperative, coalesced emission)
    __device__ static float obs_at(const St& s, int role, bool, int f) {
        return s.b[f >> 1] == ((f & 1) ? 2 - role : role + 1) ? 1.0f : 0.0f;
    }
    template <class W> __device__ static void encode(const St& s, W& w) { for (int i = 0; i < 10; i++) w.u8(s.b[i]); }
};

// ------------------------------------------------------------ Connect Four
// blob: bb0 (q0), bb1 (q1), role (16); bit = col * 7 + row, row 0 at the bottom (connect_four.py:1-80)
struct ConnectFour {
    static constexpr int A = 7, P = 2, OBS = 84;
    __device__ static int role(const St& s) { return s.b[16]; }
    __device__ static bool has_line(uint64_t bb) {
        const int sh[4] = {1, 7, 6, 8};
        for (int k = 0; k < 4; k++) {
            const uint64_t m = bb & (bb >> sh[k]);
            if (m & (m >> (2 * sh[k]))) return true;
        }
        return false;
    }
    __device__ static int height(const St& s, int col) { return __popcll(((s.q[0] | s.q[1]) >> (7 * col)) & 0x7Full); }
    __device__ static bool init(St& s, uint64_t) { s.q[0] = 0; s.q[1] = 0; s.b[16] = 0; return false; }
    __device__ static Out apply(St& s, int a, uint64_t) {
        const int mover = s.b[16];
        const uint64_t bit = 1ull << (a * 7 + height(s, a));
        s.q[mover] |= bit;
        const bool won = has_line(s.q[mover]);
        s.b[16] = (uint8_t)(1 - mover);
        if (won) return win_for(mover);
        return Out{__popcll(s.q[0] | s.q[1]) == 42, 0.0f, 0.0f};
    }
    __device__ static Mask128 mask(const St& s) {
        uint64_t m = 0;
        for (int c = 0; c < 7; c++) m |= (uint64_t)(height(s, c) < 6) << c;
        return Mask128{m, 0};
    }
    __device__ static void observe(const St& s, int role, bool, float* o) {   // (6, 7, 2), row 0 at the top
        const uint64_t mine = s.q[role], theirs = s.q[1 - role];
        float4* o4 = reinterpret_cast<float4*>(o);   // 84-float records: 16-byte aligned
#pragma unroll
        for (int i = 0; i < 42; i += 2) {   // cells i, i + 1 (row-major, row 0 at the top)
            const int b0 = (i % 7) * 7 + (5 - i / 7), b1 = ((i + 1) % 7) * 7 + (5 - (i + 1) / 7);
            o4[i / 2] = make_float4((float)((mine >> b0) & 1ull), (float)((theirs >> b0) & 1ull),
                                    (float)((mine >> b1) & 1ull), (float)((theirs >> b1) & 1ull));
        }
    }
    __device__ static float obs_at(const St& s, int role, bool, int f) {
        const int i = f >> 1, r = i / 7, c = i - 7 * (i / 7);
        return (float)((s.q[(f & 1) ? 1 - role : role] >> (c * 7 + 5 - r)) & 1ull);
    }
    template <class W> __device__ static void encode(const St& s, W& w) {
        for (int k = 0; k < 7; k++) w.u8((uint32_t)(s.q[0] >> (8 * k)) & 0xFF);
        for (int k = 0; k < 7; k++) w.u8((uint32_t)(s.q[1] >> (8 * k)) & 0xFF);
        w.u8(s.b[16]);
    }
};

// ------------------------------------------------------------ Othello
// blob: bb0 (q0), bb1 (q1), role (16), pass count (17)   (othello.py:1-150)
struct Othello {
    static constexpr int A = 65, P = 2, OBS = 128;
    static constexpr uint64_t NOT_A = 0xFEFEFEFEFEFEFEFEull, NOT_H = 0x7F7F7F7F7F7F7F7Full;
    __device__ static int role(const St& s) { return s.b[16]; }
    __device__ static uint64_t shift(uint64_t x, int d) {
        switch (d) {
            case 0: return (x << 1) & NOT_A;   // e
            case 1: return (x >> 1) & NOT_H;   // w
            case 2: return x << 8;             // s
            case 3: return x >> 8;             // n
            case 4: return (x << 9) & NOT_A;   // se
            case 5: return (x << 7) & NOT_H;   // sw
            case 6: return (x >> 7) & NOT_A;   // ne
            default: return (x >> 9) & NOT_H; // nw
        }
    }
    __device__ static uint64_t legal_moves(uint64_t mine, uint64_t theirs) {
        const uint64_t empty = ~(mine | theirs);
        uint64_t moves = 0;
        for (int d = 0; d < 8; d++) {
            uint64_t t = shift(mine, d) & theirs;
            for (int k = 0; k < 5; k++) t |= shift(t, d) & theirs;
            moves |= shift(t, d) & empty;
        }
        return moves;
    }
    __device__ static uint64_t flips_for(uint64_t bit, uint64_t mine, uint64_t theirs) {
        uint64_t flips = 0;
        for (int d = 0; d < 8; d++) {
            uint64_t ray = 0, cur = shift(bit, d);
            while (cur & theirs) { ray |= cur; cur = shift(cur, d); }
            if (cur & mine) flips |= ray;
        }
        return flips;
    }
    __device__ static Out final_rewards(const St& s) {
        const int d0 = __popcll(s.q[0]), d1 = __popcll(s.q[1]);
        if (d0 > d1) return Out{true, 1.0f, -1.0f};
        if (d1 > d0) return Out{true, -1.0f, 1.0f};
        return Out{true, 0.0f, 0.0f};
    }
    __device__ static bool init(St& s, uint64_t) {
        s.q[0] = (1ull << 28) | (1ull << 35);
        s.q[1] = (1ull << 27) | (1ull << 36);
        s.b[16] = 0; s.b[17] = 0;
        return false;
    }
    __device__ static Out apply(St& s, int a, uint64_t) {
        const int mover = s.b[16];
        s.b[16] = (uint8_t)(1 - mover);
        if (a == 64) {
            s.b[17] += 1;
            if (s.b[17] == 2) return final_rewards(s);
            return Out{false, 0.0f, 0.0f};
        }
        uint64_t mine = s.q[mover], theirs = s.q[1 - mover];
        const uint64_t bit = 1ull << a, fl = flips_for(bit, mine, theirs);
        mine |= bit | fl;
        theirs &= ~fl;
        s.q[mover] = mine; s.q[1 - mover] = theirs;
        s.b[17] = 0;
        if ((mine | theirs) == ~0ull) return final_rewards(s);
        return Out{false, 0.0f, 0.0f};
    }
    __device__ static Mask128 mask(const St& s) {   // _mask_for(side to move, other)
        const int r = s.b[16];
        const uint64_t m = legal_moves(s.q[r], s.q[1 - r]);
        return m ? Mask128{m, 0} : Mask128{0, 1};
    }
    __device__ static void observe(const St& s, int role, bool, float* o) {   // (8, 8, 2)
        const uint64_t mine = s.q[role], theirs = s.q[1 - role];
        float4* o4 = reinterpret_cast<float4*>(o);   // 128-float records: 16-byte aligned
#pragma unroll
        for (int i = 0; i < 64; i += 2)
            o4[i / 2] = make_float4((float)((mine >> i) & 1ull), (float)((theirs >> i) & 1ull),
                                    (float)((mine >> (i + 1)) & 1ull), (float)((theirs >> (i + 1)) & 1ull));
    }
    __device__ static float obs_at(const St& s, int role, bool, int f) {
        return (float)((s.q[(f & 1) ? 1 - role : role] >> (f >> 1)) & 1ull);
    }
    template <class W> __device__ static void encode(const St& s, W& w) {
        for (int k = 0; k < 8; k++) w.u8((uint32_t)(s.q[0] >> (8 * k)) & 0xFF);
        for (int k = 0; k < 8; k++) w.u8((uint32_t)(s.q[1] >> (8 * k)) & 0xFF);
        w.u8(s.b[16]);
        w.u8(s.b[17]);
    }
};

// ------------------------------------------------------------ Hex 11x11
// blob: bb0 (q0 lo, q1 hi), bb1 (q2 lo, q3 hi), move number i32 (32), swapped (36), role (37)
// (hexgame.py:1-120); 121-bit cell sets as (lo, hi) pairs.
struct U128 {   // shl / shr take 1 <= n < 128
    uint64_t lo, hi;
    __device__ U128 operator|(U128 o) const { return U128{lo | o.lo, hi | o.hi}; }
    __device__ U128 operator&(U128 o) const { return U128{lo & o.lo, hi & o.hi}; }
    __device__ U128 operator~() const { return U128{~lo, ~hi}; }
    __device__ bool any() const { return (lo | hi) != 0; }
    __device__ bool operator==(U128 o) const { return lo == o.lo && hi == o.hi; }
    __device__ U128 shl(int n) const { return n >= 64 ? U128{0, lo << (n - 64)} : U128{lo << n, (hi << n) | (lo >> (64 - n))}; }
    __device__ U128 shr(int n) const { return n >= 64 ? U128{hi >> (n - 64), 0} : U128{(lo >> n) | (hi << (64 - n)), hi >> n}; }
};

struct Hex {
    static constexpr int N = 11, CELLS = 121, SWAP = 121, A = 122, P = 2, OBS = 484;
    __device__ static U128 full() { return U128{~0ull, (1ull << (CELLS - 64)) - 1}; }
    __device__ static U128 col(int c) {   // bits r * N + c
        U128 x{0, 0};
        for (int r = 0; r < N; r++) x = x | one(r * N + c);
        return x;
    }
    __device__ static U128 one(int i) { return i < 64 ? U128{1ull << i, 0} : U128{0, 1ull << (i - 64)}; }
    __device__ static U128 neighbors(U128 x) {
        const U128 c0 = col(0), cl = col(N - 1);
        U128 out = x.shr(N);
        out = out | (x & ~cl).shr(N - 1);
        out = out | (x & ~c0).shr(1);
        out = out | (x & ~cl).shl(1);
        out = out | (x & ~c0).shl(N - 1);
        out = out | x.shl(N);
        return out & full();
    }
    __device__ static bool connected(U128 stones, U128 start, U128 goal) {
        U128 frontier = stones & start;
        if (!frontier.any()) return false;
        while (true) {
            const U128 grown = (frontier | neighbors(frontier)) & stones;
            if (grown == frontier) return false;
            if ((grown & goal).any()) return true;
            frontier = grown;
        }
    }
    __device__ static U128 bb(const St& s, int r) { return U128{s.q[2 * r], s.q[2 * r + 1]}; }
    __device__ static void set_bb(St& s, int r, U128 x) { s.q[2 * r] = x.lo; s.q[2 * r + 1] = x.hi; }
    __device__ static int move_number(const St& s) { return (int)(s.b[32] | (s.b[33] << 8) | (s.b[34] << 16) | ((uint32_t)s.b[35] << 24)); }
    __device__ static void set_move_number(St& s, int m) { for (int k = 0; k < 4; k++) s.b[32 + k] = (uint8_t)((uint32_t)m >> (8 * k)); }
    __device__ static int role(const St& s) { return s.b[37]; }
    __device__ static bool init(St& s, uint64_t) { for (int i = 0; i < 40; i++) s.b[i] = 0; return false; }
    __device__ static Out apply(St& s, int a, uint64_t) {
        const int mover = s.b[37];
        const int mn = move_number(s) + 1;
        set_move_number(s, mn);
        s.b[37] = (uint8_t)(1 - mover);
        if (a == SWAP) {
            const U128 b0 = bb(s, 0);
            const int idx = b0.hi ? 64 + 63 - __clzll(b0.hi) : 63 - __clzll(b0.lo);
            const int r = idx / N, c = idx - N * r;
            set_bb(s, 0, U128{0, 0});
            set_bb(s, 1, one(c * N + r));
            s.b[36] = 1;
            return Out{false, 0.0f, 0.0f};
        }
        U128 mine = bb(s, mover) | one(a);
        set_bb(s, mover, mine);
        bool won;
        if (mover == 0) {
            const U128 row0{(1ull << N) - 1, 0};
            const U128 rowl = row0.shl((N - 1) * N);
            won = connected(mine, row0, rowl);
        } else {
            won = connected(mine, col(0), col(N - 1));
        }
        if (won) return win_for(mover);
        return Out{false, 0.0f, 0.0f};
    }
    __device__ static Mask128 mask(const St& s) {
        const U128 m = ~(bb(s, 0) | bb(s, 1)) & full();
        return Mask128{m.lo, m.hi | (move_number(s) == 1 ? (1ull << (SWAP - 64)) : 0ull)};
    }
    __device__ static void observe(const St& s, int role, bool terminal, float* o) {   // (11, 11, 4)
        const U128 mine = bb(s, role), theirs = bb(s, 1 - role);
        const float swap = (!terminal && move_number(s) == 1) ? 1.0f : 0.0f;
        float4* o4 = reinterpret_cast<float4*>(o);   // one float4 per cell (484-float records: aligned)
        for (int i = 0; i < CELLS; i++) {
            const bool m = i < 64 ? (mine.lo >> i) & 1ull : (mine.hi >> (i - 64)) & 1ull;
            const bool t = i < 64 ? (theirs.lo >> i) & 1ull : (theirs.hi >> (i - 64)) & 1ull;
            o4[i] = make_float4(m ? 1.0f : 0.0f, t ? 1.0f : 0.0f, (float)role, swap);
        }
    }
    __device__ static float obs_at(const St& s, int role, bool terminal, int f) {
        const int i = f >> 2, ch = f & 3;
        if (ch == 2) return (float)role;
        if (ch == 3) return (!terminal && move_number(s) == 1) ? 1.0f : 0.0f;
        const U128 x = bb(s, ch == 0 ? role : 1 - role);
        return (float)(i < 64 ? (x.lo >> i) & 1ull : (x.hi >> (i - 64)) & 1ull);
    }
    template <class W> __device__ static void encode(const St& s, W& w) {
        for (int k = 0; k < 32; k++) w.u8(s.b[k]);   // bb0, bb1 as 16-byte little-endian integers
        w.u8(s.b[37]);
        w.u8(s.b[32]);   // move_number & 0xFF
        w.u8(s.b[36]);
    }
};

// ------------------------------------------------------------ 2048
// blob: board exponents [16], score u64 (q2)   (play2048.py:1-134)
struct Play2048 {
    static constexpr int A = 4, P = 1, OBS = 496;
    __device__ static int role(const St&) { return 0; }
    __device__ static int line_cell(int dir, int l, int j) {   // movement side first
        switch (dir) {
            case 0: return 4 * l + j;         // LEFT
            case 1: return 4 * j + l;         // UP
            case 2: return 4 * l + (3 - j);   // RIGHT
            default: return 4 * (3 - j) + l; // DOWN
        }
    }
    // slide without spawning (play2048.py:35-66); returns the merged-tile sum
    __device__ static uint32_t slide(const uint8_t* in, int dir, uint8_t* out) {
        uint32_t reward = 0;
        for (int l = 0; l < 4; l++) {
            uint8_t o[4] = {0, 0, 0, 0};
            int n = 0, open = -1;
            for (int j = 0; j < 4; j++) {
                const uint8_t v = in[line_cell(dir, l, j)];
                if (!v) continue;
                if (open >= 0 && o[open] == v) { o[open] = (uint8_t)(v + 1); reward += 1u << (v + 1); open = -1; }
                else { o[n] = v; open = n; n++; }
            }
            for (int j = 0; j < 4; j++) out[line_cell(dir, l, j)] = o[j];
        }
        return reward;
    }
    __device__ static void spawn(uint8_t* board, uint64_t key) {   // play2048.py:69-75
        int empties = 0;
        for (int i = 0; i < 16; i++) empties += board[i] == 0;
        int pick = (int)umod_small(child(key, 0), (uint32_t)empties);
        const uint8_t e = (child(key, 1) % 10ull) == 9ull ? 2 : 1;
        for (int i = 0; i < 16; i++)
            if (board[i] == 0 && pick-- == 0) { board[i] = e; break; }
    }
    __device__ static uint32_t dirs(const St& s) {
        uint32_t m = 0;
        for (int d = 0; d < 4; d++) {
            uint8_t o[16];
            slide(s.b, d, o);
            bool ch = false;
            for (int i = 0; i < 16; i++) ch |= o[i] != s.b[i];
            m |= (uint32_t)ch << d;
        }
        return m;
    }
    __device__ static bool init(St& s, uint64_t key) {   // _init_core: two spawns from key.child(0), key.child(1)
        for (int i = 0; i < 16; i++) s.b[i] = 0;
        s.q[2] = 0;
        spawn(s.b, child(key, 0));
        spawn(s.b, child(key, 1));
        return dirs(s) == 0;
    }
    __device__ static Out apply(St& s, int a, uint64_t key) {
        uint8_t o[16];
        const uint32_t reward = slide(s.b, a, o);
        for (int i = 0; i < 16; i++) s.b[i] = o[i];
        spawn(s.b, key);
        s.q[2] += reward;
        return Out{dirs(s) == 0, (float)reward, 0.0f};
    }
    __device__ static Mask128 mask(const St& s) { return Mask128{dirs(s), 0}; }
    __device__ static void observe(const St& s, int, bool, float* o) {   // (4, 4, 31) one-hot exponents
        float4* o4 = reinterpret_cast<float4*>(o);   // 496-float records: 16-byte aligned
        for (int j = 0; j < 124; j++) {   // float 4j + t is cell (4j + t) / 31, plane (4j + t) % 31
            float v[4];
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int f = 4 * j + t, cell = f / 31;
                v[t] = s.b[cell] == f - 31 * cell + 1 ? 1.0f : 0.0f;
            }
            o4[j] = make_float4(v[0], v[1], v[2], v[3]);
        }
    }
    __device__ static float obs_at(const St& s, int, bool, int f) {
        const int cell = f / 31;
        return s.b[cell] == f - 31 * cell + 1 ? 1.0f : 0.0f;
    }
    template <class W> __device__ static void encode(const St& s, W& w) {
        for (int i = 0; i < 16; i++) w.u8(s.b[i]);
        w.u64(s.q[2]);
    }
};

// ------------------------------------------------------------ Kuhn poker
// blob: hands[2] (0,1), history[4] (2..5), history length (6), extra[2] (7,8), role (9)
// actions CALL 0, BET 1, FOLD 2, CHECK 3   (kuhn_poker.py:1-76)
struct Kuhn {
    static constexpr int A = 4, P = 2, OBS = 7;
    __device__ static int role(const St& s) { return s.b[9]; }
    __device__ static bool init(St& s, uint64_t key) {
        int deal[3];
        permutation(key, 3, deal);
        for (int i = 0; i < 10; i++) s.b[i] = 0;
        s.b[0] = (uint8_t)deal[0]; s.b[1] = (uint8_t)deal[1];
        return false;
    }
    __device__ static Out showdown(const St& s, float stake) {
        return s.b[0] > s.b[1] ? Out{true, stake, -stake} : Out{true, -stake, stake};
    }
    __device__ static Out apply(St& s, int a, uint64_t) {
        const int mover = s.b[9], hl = s.b[6];
        const bool prior_check = hl == 1 && s.b[2] == 3;
        s.b[2 + hl] = (uint8_t)a;
        s.b[6] = (uint8_t)(hl + 1);
        s.b[9] = (uint8_t)(1 - mover);
        if (a == 1) { s.b[7 + mover] = 1; return Out{false, 0.0f, 0.0f}; }
        if (a == 3) return prior_check ? showdown(s, 1.0f) : Out{false, 0.0f, 0.0f};
        if (a == 0) { s.b[7 + mover] = 1; return showdown(s, 2.0f); }
        return mover == 0 ? Out{true, -1.0f, 1.0f} : Out{true, 1.0f, -1.0f};   // fold
    }
    __device__ static Mask128 mask(const St& s) {   // facing a bet: call / fold, else bet / check
        const int hl = s.b[6];
        const bool facing = hl > 0 && s.b[2 + hl - 1] == 1;
        return Mask128{facing ? 0x5ull : 0xAull, 0};
    }
    __device__ static void observe(const St& s, int role, bool, float* o) {
        for (int i = 0; i < 7; i++) o[i] = 0.0f;
        o[s.b[role]] = 1.0f;
        o[3 + s.b[7 + role]] = 1.0f;
        o[5 + s.b[7 + 1 - role]] = 1.0f;
    }
    __device__ static float obs_at(const St& s, int role, bool, int f) {
        if (f < 3) return f == s.b[role] ? 1.0f : 0.0f;
        if (f < 5) return f - 3 == s.b[7 + role] ? 1.0f : 0.0f;
        return f - 5 == s.b[7 + 1 - role] ? 1.0f : 0.0f;
    }
    template <class W> __device__ static void encode(const St& s, W& w) {
        w.u8(s.b[0]); w.u8(s.b[1]);
        for (int i = 0; i < s.b[6]; i++) w.u8(s.b[2 + i]);
        w.u8(0xFF);
        w.u8(s.b[7]); w.u8(s.b[8]);
    }
};

// ------------------------------------------------------------ Leduc hold'em
// blob: hands (0,1), public + 1 (2), round (3), raises (4), committed (5,6), acted (7), role (8)
// actions CALL 0, RAISE 1, FOLD 2   (leduc_holdem.py:1-125)
struct Leduc {
    static constexpr int A = 3, P = 2, OBS = 34;
    __device__ static int role(const St& s) { return s.b[8]; }
    __device__ static bool init(St& s, uint64_t key) {
        int deal[6];
        permutation(key, 6, deal);
        for (int i = 0; i < 10; i++) s.b[i] = 0;
        s.b[0] = (uint8_t)(deal[0] / 2); s.b[1] = (uint8_t)(deal[1] / 2);   // deck J J Q Q K K
        s.b[3] = 1; s.b[5] = 1; s.b[6] = 1;
        return false;
    }
    __device__ static Out stake_to(int winner, float stake) {
        return winner == 0 ? Out{true, stake, -stake} : Out{true, -stake, stake};
    }
    __device__ static Out apply(St& s, int a, uint64_t key) {
        const int mover = s.b[8];
        const int mx = s.b[5] > s.b[6] ? s.b[5] : s.b[6];
        if (a == 2) {   // fold: the other player wins the folder's commitment
            s.b[8] = (uint8_t)(1 - mover);
            return stake_to(1 - mover, (float)s.b[5 + mover]);
        }
        if (a == 0) {
            s.b[5 + mover] = (uint8_t)mx;
            if (s.b[7] >= 1) {
                if (s.b[3] == 2) {   // showdown
                    s.b[8] = (uint8_t)(1 - mover);
                    const int h0 = s.b[0], h1 = s.b[1], pub = (int)s.b[2] - 1;
                    int winner;
                    if (h0 == pub) winner = 0;
                    else if (h1 == pub) winner = 1;
                    else if (h0 != h1) winner = h0 > h1 ? 0 : 1;
                    else return Out{true, 0.0f, 0.0f};
                    return stake_to(winner, (float)s.b[5 + 1 - winner]);
                }
                // public card: the remaining deck (J J Q Q K K minus both hands) at key % 4
                int deck[6] = {0, 0, 1, 1, 2, 2}, m = 6;
                for (int h = 0; h < 2; h++) {
                    for (int j = 0; j < m; j++)
                        if (deck[j] == s.b[h]) { for (int q = j; q < m - 1; q++) deck[q] = deck[q + 1]; m--; break; }
                }
                s.b[2] = (uint8_t)(deck[key % 4ull] + 1);
                s.b[3] = 2; s.b[4] = 0; s.b[7] = 0; s.b[8] = 0;
                return Out{false, 0.0f, 0.0f};
            }
            s.b[7] = 1;
            s.b[8] = (uint8_t)(1 - mover);
            return Out{false, 0.0f, 0.0f};
        }
        const int amount = s.b[3] == 1 ? 2 : 4;   // raise
        s.b[5 + mover] = (uint8_t)(mx + amount);
        s.b[4] += 1;
        s.b[7] += 1;
        s.b[8] = (uint8_t)(1 - mover);
        return Out{false, 0.0f, 0.0f};
    }
    __device__ static Mask128 mask(const St& s) { return Mask128{s.b[4] < 2 ? 0x7ull : 0x5ull, 0}; }
    __device__ static void observe(const St& s, int role, bool, float* o) {
        for (int i = 0; i < 34; i++) o[i] = 0.0f;
        o[s.b[role]] = 1.0f;
        if (s.b[2]) o[3 + s.b[2] - 1] = 1.0f;
        o[6 + s.b[5 + role]] = 1.0f;
        o[20 + s.b[5 + 1 - role]] = 1.0f;
    }
    __device__ static float obs_at(const St& s, int role, bool, int f) {
        if (f < 3) return f == s.b[role] ? 1.0f : 0.0f;
        if (f < 6) return (s.b[2] && f - 3 == s.b[2] - 1) ? 1.0f : 0.0f;
        if (f < 20) return f - 6 == s.b[5 + role] ? 1.0f : 0.0f;
        return f - 20 == s.b[5 + 1 - role] ? 1.0f : 0.0f;
    }
    template <class W> __device__ static void encode(const St& s, W& w) { for (int i = 0; i < 9; i++) w.u8(s.b[i]); }
};

}  // namespace small
