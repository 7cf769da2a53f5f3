/* ORACLE (test infrastructure only) -- chess, CPU engine.
 *
 * The reference has NO chess engine (reserved GameSpec("chess", 2, (8,8,119),
 * 4672), pkg/src/boardbatch/games/__init__.py:23; tests assert it raises,
 * test_core.py:36-42). This oracle restates the rules and encodings the
 * paper specifies (AlphaZero 8x8x119 observation and
 * 64x73 action encoding, +1/-1/0 rewards) with the env-core contract of
 * core.py:192-243 and the decisions recorded in DESIGN.md §3.3. It is
 * pinned by perft known-answer tests (tests/test_oracle_chess.py), NOT by
 * the reference: parity against the reference is "unpinned" for chess.
 *
 * Deliberately simple and independent of the CUDA kernel: 8x8 mailbox,
 * pseudo-legal generation + make/undo + "is my king attacked" legality.
 * Only tests/, __graft_entry__.smoke() and bench.py may load this code.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include "orc_rng.h"

#define CH_A 4672
#define CH_OBS (8 * 8 * 119)
#define CH_RING 128

enum { EMPTY = 0, P = 1, N = 2, B = 3, R = 4, Q = 5, K = 6 };
#define COLOR(pc) ((pc) >> 3)          /* 0 white, 1 black */
#define TYPE(pc) ((pc) & 7)
#define MK(c, t) ((uint8_t)(((c) << 3) | (t)))

typedef struct {
    uint8_t sq[64];   /* a1 = 0, b1 = 1, ..., h8 = 63 */
    uint8_t stm;      /* side to move: 0 white (role 0), 1 black */
    uint8_t castle;   /* 1 W-O-O, 2 W-O-O-O, 4 B-O-O, 8 B-O-O-O */
    int8_t ep;        /* en-passant target square or -1 */
    uint8_t halfmove;
} cpos;

typedef struct { uint8_t from, to, promo; } cmove;

typedef struct {
    uint8_t board[64];
    uint8_t stm, castle;
    int8_t ep_eff;     /* ep square only if an en-passant capture is legal */
    uint8_t rep;       /* prior occurrences (capped at 2) */
} hentry;

typedef struct {
    cpos pos;
    hentry ring[CH_RING];   /* ring[ply % CH_RING], ply 0 = initial position */
    uint8_t mask[CH_A];
    uint8_t terminal, truncated;
    float role_rewards[2];
    int32_t step_count;
    int8_t p2r[2];
    uint8_t rep;
} ch_env;

typedef struct {
    int64_t n;
    int max_steps;
    ch_env* env;
} orc_chess;

static const int KN_DR[8] = {2, 1, -1, -2, -2, -1, 1, 2};
static const int KN_DF[8] = {1, 2, 2, 1, -1, -2, -2, -1};
static const int DIR_DR[8] = {1, 1, 0, -1, -1, -1, 0, 1};   /* N NE E SE S SW W NW */
static const int DIR_DF[8] = {0, 1, 1, 1, 0, -1, -1, -1};

static inline int on(int r, int f) { return r >= 0 && r < 8 && f >= 0 && f < 8; }

/* Is square s attacked by side `by`? */
static int attacked(const cpos* p, int s, int by) {
    int r = s >> 3, f = s & 7;
    /* pawns: a pawn of `by` attacks diagonally forward */
    int pr = by == 0 ? r - 1 : r + 1;
    for (int df = -1; df <= 1; df += 2)
        if (on(pr, f + df) && p->sq[pr * 8 + f + df] == MK(by, P)) return 1;
    for (int k = 0; k < 8; k++) {
        int rr = r + KN_DR[k], ff = f + KN_DF[k];
        if (on(rr, ff) && p->sq[rr * 8 + ff] == MK(by, N)) return 1;
    }
    for (int d = 0; d < 8; d++) {
        int rr = r + DIR_DR[d], ff = f + DIR_DF[d];
        if (on(rr, ff) && p->sq[rr * 8 + ff] == MK(by, K)) return 1;
        int diag = DIR_DR[d] != 0 && DIR_DF[d] != 0;
        while (on(rr, ff)) {
            uint8_t pc = p->sq[rr * 8 + ff];
            if (pc) {
                if (COLOR(pc) == by && (TYPE(pc) == Q || TYPE(pc) == (diag ? B : R))) return 1;
                break;
            }
            rr += DIR_DR[d]; ff += DIR_DF[d];
        }
    }
    return 0;
}

static int king_sq(const cpos* p, int side) {
    for (int s = 0; s < 64; s++) if (p->sq[s] == MK(side, K)) return s;
    return -1;
}

static int in_check(const cpos* p, int side) {
    int k = king_sq(p, side);
    return k >= 0 && attacked(p, k, 1 - side);
}

static void make(cpos* p, cmove m) {
    uint8_t pc = p->sq[m.from], cap = p->sq[m.to];
    int side = COLOR(pc), t = TYPE(pc);
    int reset_clock = t == P || cap != EMPTY;
    if (t == P && m.to == p->ep && cap == EMPTY && (m.from & 7) != (m.to & 7)) {
        int victim = side == 0 ? m.to - 8 : m.to + 8;   /* en passant */
        p->sq[victim] = EMPTY;
    }
    p->sq[m.to] = m.promo ? MK(side, m.promo) : pc;
    p->sq[m.from] = EMPTY;
    if (t == K && abs((m.to & 7) - (m.from & 7)) == 2) {   /* castling: move the rook */
        int rank = m.from & ~7;
        if ((m.to & 7) == 6) { p->sq[rank + 5] = p->sq[rank + 7]; p->sq[rank + 7] = EMPTY; }
        else { p->sq[rank + 3] = p->sq[rank + 0]; p->sq[rank + 0] = EMPTY; }
    }
    /* castling rights: king or rook moved, rook captured */
    static const uint8_t clear_on[64] = {
        [0] = 2, [4] = 3, [7] = 1, [56] = 8, [60] = 12, [63] = 4};
    p->castle &= (uint8_t)~(clear_on[m.from] | clear_on[m.to]);
    p->ep = -1;
    if (t == P && abs(m.to - m.from) == 16) p->ep = (int8_t)((m.from + m.to) / 2);
    p->halfmove = reset_clock ? 0 : (uint8_t)(p->halfmove + 1);
    p->stm ^= 1;
}

/* Pseudo-legal moves of the side to move. */
static int gen_pseudo(const cpos* p, cmove* out) {
    int n = 0, side = p->stm;
    for (int s = 0; s < 64; s++) {
        uint8_t pc = p->sq[s];
        if (!pc || COLOR(pc) != side) continue;
        int r = s >> 3, f = s & 7, t = TYPE(pc);
        if (t == P) {
            int dr = side == 0 ? 1 : -1, last = side == 0 ? 7 : 0, start = side == 0 ? 1 : 6;
            int r1 = r + dr;
            if (on(r1, f) && !p->sq[r1 * 8 + f]) {
                if (r1 == last) { for (int pr = Q; pr >= N; pr--) out[n++] = (cmove){(uint8_t)s, (uint8_t)(r1 * 8 + f), (uint8_t)pr}; }
                else {
                    out[n++] = (cmove){(uint8_t)s, (uint8_t)(r1 * 8 + f), 0};
                    int r2 = r + 2 * dr;
                    if (r == start && !p->sq[r2 * 8 + f]) out[n++] = (cmove){(uint8_t)s, (uint8_t)(r2 * 8 + f), 0};
                }
            }
            for (int df = -1; df <= 1; df += 2) {
                if (!on(r1, f + df)) continue;
                int to = r1 * 8 + f + df;
                uint8_t c = p->sq[to];
                if ((c && COLOR(c) != side) || to == p->ep) {
                    if (r1 == last) { for (int pr = Q; pr >= N; pr--) out[n++] = (cmove){(uint8_t)s, (uint8_t)to, (uint8_t)pr}; }
                    else out[n++] = (cmove){(uint8_t)s, (uint8_t)to, 0};
                }
            }
        } else if (t == N) {
            for (int k = 0; k < 8; k++) {
                int rr = r + KN_DR[k], ff = f + KN_DF[k];
                if (!on(rr, ff)) continue;
                uint8_t c = p->sq[rr * 8 + ff];
                if (!c || COLOR(c) != side) out[n++] = (cmove){(uint8_t)s, (uint8_t)(rr * 8 + ff), 0};
            }
        } else {
            int d0 = t == B ? 1 : 0, step = (t == B || t == R) ? 2 : 1;
            int slide = t != K;
            for (int d = d0; d < 8; d += step) {
                int rr = r + DIR_DR[d], ff = f + DIR_DF[d];
                while (on(rr, ff)) {
                    uint8_t c = p->sq[rr * 8 + ff];
                    if (c && COLOR(c) == side) break;
                    out[n++] = (cmove){(uint8_t)s, (uint8_t)(rr * 8 + ff), 0};
                    if (c || !slide) break;
                    rr += DIR_DR[d]; ff += DIR_DF[d];
                }
            }
            if (t == K) {   /* castling */
                int rank = side == 0 ? 0 : 56;
                int kbit = side == 0 ? 1 : 4, qbit = side == 0 ? 2 : 8;
                if (s == rank + 4 && !attacked(p, s, 1 - side)) {
                    if ((p->castle & kbit) && p->sq[rank + 7] == MK(side, R) && !p->sq[rank + 5] && !p->sq[rank + 6] &&
                        !attacked(p, rank + 5, 1 - side) && !attacked(p, rank + 6, 1 - side))
                        out[n++] = (cmove){(uint8_t)s, (uint8_t)(rank + 6), 0};
                    if ((p->castle & qbit) && p->sq[rank + 0] == MK(side, R) && !p->sq[rank + 1] && !p->sq[rank + 2] &&
                        !p->sq[rank + 3] && !attacked(p, rank + 3, 1 - side) && !attacked(p, rank + 2, 1 - side))
                        out[n++] = (cmove){(uint8_t)s, (uint8_t)(rank + 2), 0};
                }
            }
        }
    }
    return n;
}

static int gen_legal(const cpos* p, cmove* out) {
    cmove tmp[256];
    int n = gen_pseudo(p, tmp), k = 0;
    for (int i = 0; i < n; i++) {
        cpos q = *p;
        make(&q, tmp[i]);
        if (!in_check(&q, p->stm)) out[k++] = tmp[i];
    }
    return k;
}

/* AlphaZero 64x73 action index in the mover's frame. */
static int action_of(int stm, cmove m) {
    int fl = stm ? 56 : 0;
    int from = m.from ^ fl, to = m.to ^ fl;
    int dr = (to >> 3) - (from >> 3), df = (to & 7) - (from & 7);
    int plane = -1;
    if (m.promo && m.promo != Q) {
        int pi = m.promo == N ? 0 : m.promo == B ? 1 : 2;
        plane = 64 + 3 * pi + (df + 1);
    } else {
        for (int k = 0; k < 8; k++) if (KN_DR[k] == dr && KN_DF[k] == df) plane = 56 + k;
        if (plane < 0) {
            int dist = abs(dr) > abs(df) ? abs(dr) : abs(df);
            int sr = (dr > 0) - (dr < 0), sf = (df > 0) - (df < 0);
            for (int d = 0; d < 8; d++) if (DIR_DR[d] == sr && DIR_DF[d] == sf) plane = d * 7 + dist - 1;
        }
    }
    return from * 73 + plane;
}

static const uint8_t START[64] = {
    MK(0, R), MK(0, N), MK(0, B), MK(0, Q), MK(0, K), MK(0, B), MK(0, N), MK(0, R),
    MK(0, P), MK(0, P), MK(0, P), MK(0, P), MK(0, P), MK(0, P), MK(0, P), MK(0, P),
    0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
    MK(1, P), MK(1, P), MK(1, P), MK(1, P), MK(1, P), MK(1, P), MK(1, P), MK(1, P),
    MK(1, R), MK(1, N), MK(1, B), MK(1, Q), MK(1, K), MK(1, B), MK(1, N), MK(1, R)};

static int insufficient(const cpos* p) {
    int minors = 0, bishops_light = 0, bishops_dark = 0, knights = 0;
    for (int s = 0; s < 64; s++) {
        int t = TYPE(p->sq[s]);
        if (!p->sq[s] || t == K) continue;
        if (t == P || t == R || t == Q) return 0;
        minors++;
        if (t == N) knights++;
        else if ((((s >> 3) + (s & 7)) & 1)) bishops_light++;
        else bishops_dark++;
    }
    if (minors <= 1) return 1;
    if (knights == 0 && (bishops_light == 0 || bishops_dark == 0)) return 1;
    return 0;
}

/* Evaluate the new position: legal mask, repetition, terminal, rewards. */
static void settle(orc_chess* g, ch_env* e) {
    cmove mv[256];
    int n = gen_legal(&e->pos, mv);
    memset(e->mask, 0, CH_A);
    int ep_legal = 0;
    for (int i = 0; i < n; i++) {
        e->mask[action_of(e->pos.stm, mv[i])] = 1;
        if (TYPE(e->pos.sq[mv[i].from]) == P && mv[i].to == e->pos.ep) ep_legal = 1;
    }
    /* repetition: identical (board, stm, castling, legal-ep) within the halfmove window */
    hentry cur;
    memcpy(cur.board, e->pos.sq, 64);
    cur.stm = e->pos.stm; cur.castle = e->pos.castle; cur.ep_eff = ep_legal ? e->pos.ep : -1;
    int reps = 0;
    for (int back = 2; back <= e->pos.halfmove && back <= e->step_count; back += 2) {
        const hentry* h = &e->ring[(e->step_count - back) % CH_RING];
        if (h->stm == cur.stm && h->castle == cur.castle && h->ep_eff == cur.ep_eff &&
            !memcmp(h->board, cur.board, 64)) reps++;
    }
    cur.rep = (uint8_t)(reps > 2 ? 2 : reps);
    e->ring[e->step_count % CH_RING] = cur;
    e->rep = cur.rep;
    e->terminal = 0;
    e->role_rewards[0] = e->role_rewards[1] = 0.0f;
    if (n == 0) {
        e->terminal = 1;
        if (in_check(&e->pos, e->pos.stm)) {
            e->role_rewards[e->pos.stm] = -1.0f;
            e->role_rewards[1 - e->pos.stm] = 1.0f;
        }
    } else if (insufficient(&e->pos) || e->pos.halfmove >= 100 || reps >= 2) {
        e->terminal = 1;
    }
    if (e->terminal) memset(e->mask, 0, CH_A);
}

static void env_init(orc_chess* g, ch_env* e, uint64_t key) {
    uint64_t c = orc_child(key, 0) % 2;
    e->p2r[0] = (int8_t)c; e->p2r[1] = (int8_t)(1 - c);
    memcpy(e->pos.sq, START, 64);
    e->pos.stm = 0; e->pos.castle = 15; e->pos.ep = -1; e->pos.halfmove = 0;
    e->step_count = 0; e->truncated = 0;
    settle(g, e);
}

static void env_apply(orc_chess* g, ch_env* e, int action) {
    cmove mv[256];
    int n = gen_legal(&e->pos, mv);
    for (int i = 0; i < n; i++) {
        if (action_of(e->pos.stm, mv[i]) == action) { make(&e->pos, mv[i]); break; }
    }
    e->step_count += 1;
    settle(g, e);
}

orc_chess* orc_chess_new(int64_t n, int max_steps) {
    orc_chess* g = (orc_chess*)calloc(1, sizeof(orc_chess));
    g->n = n; g->max_steps = max_steps;
    g->env = (ch_env*)calloc((size_t)n, sizeof(ch_env));
    return g;
}

void orc_chess_free(orc_chess* g) { if (g) { free(g->env); free(g); } }

void orc_chess_init(orc_chess* g, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) env_init(g, &g->env[i], orc_slot_key(slot_keys, key_state, slot0, i));
}

int64_t orc_chess_step(orc_chess* g, const int64_t* actions, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    for (int64_t i = 0; i < g->n; i++) {
        ch_env* e = &g->env[i];
        if (e->terminal || e->truncated) continue;
        int64_t a = actions[i];
        if (a < 0 || a >= CH_A || !e->mask[a]) return i;
    }
    #pragma omp parallel for schedule(dynamic, 8)
    for (int64_t i = 0; i < g->n; i++) {
        ch_env* e = &g->env[i];
        uint64_t k = orc_slot_key(slot_keys, key_state, slot0, i);
        if (e->terminal || e->truncated) { env_init(g, e, k); continue; }
        env_apply(g, e, (int)actions[i]);
        e->truncated = (uint8_t)(!e->terminal && e->step_count >= g->max_steps);
        if (e->truncated) memset(e->mask, 0, CH_A);
    }
    return -1;
}

/* Observation (AlphaZero planes) for `role` (0 white, 1 black):
 * obs[rank'][file][plane], rank' = rank seen from `role` (0 = own back rank).
 * planes 14t..14t+13 for history step t (0 = current): own P N B R Q K,
 * opponent P N B R Q K, repetition >= 1, repetition >= 2; then 112 colour,
 * 113 step_count/512, 114-115 own O-O/O-O-O, 116-117 opponent's, 118 halfmove/100. */
void orc_chess_observe(const orc_chess* g, int64_t i, int role, float* obs) {
    const ch_env* e = &g->env[i];
    memset(obs, 0, sizeof(float) * CH_OBS);
    int fl = role ? 56 : 0;
    for (int t = 0; t < 8; t++) {
        int ply = e->step_count - t;
        if (ply < 0) break;
        const hentry* h = &e->ring[ply % CH_RING];
        for (int s = 0; s < 64; s++) {
            uint8_t pc = h->board[s];
            if (!pc) continue;
            int v = s ^ fl;
            int plane = 14 * t + (COLOR(pc) == role ? 0 : 6) + TYPE(pc) - 1;
            obs[v * 119 + plane] = 1.0f;
        }
        for (int v = 0; v < 64; v++) {
            if (h->rep >= 1) obs[v * 119 + 14 * t + 12] = 1.0f;
            if (h->rep >= 2) obs[v * 119 + 14 * t + 13] = 1.0f;
        }
    }
    int own_k = role ? 4 : 1, own_q = role ? 8 : 2, opp_k = role ? 1 : 4, opp_q = role ? 2 : 8;
    for (int v = 0; v < 64; v++) {
        float* o = obs + v * 119;
        o[112] = (float)role;
        o[113] = (float)e->step_count / 512.0f;
        o[114] = (e->pos.castle & own_k) ? 1.0f : 0.0f;
        o[115] = (e->pos.castle & own_q) ? 1.0f : 0.0f;
        o[116] = (e->pos.castle & opp_k) ? 1.0f : 0.0f;
        o[117] = (e->pos.castle & opp_q) ? 1.0f : 0.0f;
        o[118] = (float)e->pos.halfmove / 100.0f;
    }
}

void orc_chess_columns(const orc_chess* g, float* obs, uint8_t* mask, float* rewards, uint8_t* term,
                       uint8_t* trunc, int32_t* cur, int32_t* step_count, int8_t* p2r) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) {
        const ch_env* e = &g->env[i];
        if (mask) memcpy(mask + i * CH_A, e->mask, CH_A);
        if (rewards) {
            float r0 = 0.0f, r1 = 0.0f;
            if (!e->truncated && (e->role_rewards[0] != 0.0f || e->role_rewards[1] != 0.0f)) {
                r0 = e->role_rewards[e->p2r[0]];
                r1 = e->role_rewards[e->p2r[1]];
            }
            rewards[2 * i] = r0; rewards[2 * i + 1] = r1;
        }
        if (term) term[i] = e->terminal;
        if (trunc) trunc[i] = e->truncated;
        if (cur) cur[i] = e->p2r[0] == e->pos.stm ? 0 : 1;
        if (step_count) step_count[i] = e->step_count;
        if (p2r) { p2r[2 * i] = e->p2r[0]; p2r[2 * i + 1] = e->p2r[1]; }
        if (obs) orc_chess_observe(g, i, e->pos.stm, obs + (size_t)i * CH_OBS);
    }
}

/* encode: board[64] + stm + castle + ep + halfmove + rep. */
int orc_chess_encode(const orc_chess* g, int64_t i, uint8_t* buf) {
    const ch_env* e = &g->env[i];
    memcpy(buf, e->pos.sq, 64);
    buf[64] = e->pos.stm; buf[65] = e->pos.castle; buf[66] = (uint8_t)e->pos.ep;
    buf[67] = e->pos.halfmove; buf[68] = e->rep;
    return 69;
}

/* ---------------- perft (known-answer tests) ---------------- */
static int parse_fen(const char* fen, cpos* p) {
    memset(p, 0, sizeof(*p));
    p->ep = -1;
    int r = 7, f = 0;
    const char* c = fen;
    for (; *c && *c != ' '; c++) {
        if (*c == '/') { r--; f = 0; continue; }
        if (*c >= '1' && *c <= '8') { f += *c - '0'; continue; }
        int color = (*c >= 'a') ? 1 : 0;
        int t = 0;
        switch (*c | 32) { case 'p': t = P; break; case 'n': t = N; break; case 'b': t = B; break;
                           case 'r': t = R; break; case 'q': t = Q; break; case 'k': t = K; break; default: return -1; }
        p->sq[r * 8 + f++] = MK(color, t);
    }
    if (*c) c++;
    p->stm = *c == 'b';
    while (*c && *c != ' ') c++;
    if (*c) c++;
    for (; *c && *c != ' '; c++) {
        if (*c == 'K') p->castle |= 1; else if (*c == 'Q') p->castle |= 2;
        else if (*c == 'k') p->castle |= 4; else if (*c == 'q') p->castle |= 8;
    }
    if (*c) c++;
    if (*c && *c != '-') { p->ep = (int8_t)((c[1] - '1') * 8 + (c[0] - 'a')); }
    while (*c && *c != ' ') c++;
    if (*c) c++;
    if (*c >= '0' && *c <= '9') p->halfmove = (uint8_t)atoi(c);
    return 0;
}

static uint64_t perft(const cpos* p, int depth) {
    cmove mv[256];
    int n = gen_legal(p, mv);
    if (depth == 1) return (uint64_t)n;
    uint64_t total = 0;
    for (int i = 0; i < n; i++) {
        cpos q = *p;
        make(&q, mv[i]);
        total += perft(&q, depth - 1);
    }
    return total;
}

uint64_t orc_chess_perft(const char* fen, int depth) {
    cpos p;
    if (parse_fen(fen, &p) != 0) return 0;
    if (depth <= 0) return 1;
    return perft(&p, depth);
}

/* Test hook: load a FEN into slot i (history reset) and settle it. */
int orc_chess_set_fen(orc_chess* g, int64_t i, const char* fen) {
    ch_env* e = &g->env[i];
    if (parse_fen(fen, &e->pos) != 0) return -1;
    e->step_count = 0; e->terminal = 0; e->truncated = 0;
    settle(g, e);
    return 0;
}
