/* ORACLE (test infrastructure only) -- shogi, CPU engine.
 *
 * The reference has NO shogi engine (reserved GameSpec("shogi", 2, (9,9,119),
 * 2187), pkg/src/boardbatch/games/__init__.py:31). This oracle restates the
 * rules and encodings of PAPER.md:1278-1354 (dlshogi-style 119-plane
 * observation, 81 x 27 actions incl. 7 drops, four-fold repetition draw, no
 * stalemate) with the env-core contract of core.py:192-243 and the
 * decisions in DESIGN.md §3.4. Pinned by perft known-answer tests
 * (tests/test_oracle_shogi.py); parity against the reference is "unpinned".
 *
 * Simple mailbox engine working in the MOVER'S FRAME (Black as is, White
 * rotated 180 degrees), pseudo-legal generation + make + king-attack test;
 * independent of the CUDA kernel. Only tests/, __graft_entry__.smoke() and
 * bench.py may load this code.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "orc_rng.h"

#define SG_A 2187
#define SG_OBS (9 * 9 * 119)

enum { E = 0, FU = 1, KY, KE, GI, KI, KA, HI, OU, TO, NY, NK, NG, UM, RY };
#define SCOLOR(pc) ((pc) >> 4)
#define STYPE(pc) ((pc) & 15)
#define SMK(c, t) ((uint8_t)(((c) << 4) | (t)))

typedef struct {
    uint8_t sq[81];      /* absolute: r*9+c, r=0 top (White's back rank), c=0 left (9-file) */
    uint8_t hand[2][7];  /* FU KY KE GI KI KA HI */
    uint8_t stm;
} spos;

typedef struct { int8_t from; uint8_t to; uint8_t promo; uint8_t drop; } smove;   /* drop: hand index+1 */

typedef struct {
    spos pos;
    uint64_t* hist;      /* position keys by ply */
    uint8_t mask[SG_A];
    uint8_t terminal, truncated, rep, in_check;
    float role_rewards[2];
    int32_t step_count;
    int8_t p2r[2];
} sg_env;

typedef struct {
    int64_t n;
    int max_steps;
    sg_env* env;
} orc_shogi;

/* movement offsets in the mover's frame (forward = row - 1) */
static const int8_t GOLD_D[6][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, 0}};
static const int8_t SILVER_D[5][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {1, -1}, {1, 1}};
static const int8_t KING_D[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
static const int8_t ORTH[4][2] = {{-1, 0}, {0, -1}, {0, 1}, {1, 0}};
static const int8_t DIAG[4][2] = {{-1, -1}, {-1, 1}, {1, -1}, {1, 1}};

static inline int son(int r, int c) { return r >= 0 && r < 9 && c >= 0 && c < 9; }
/* mover-frame square <-> absolute square */
static inline int fr(int side, int s) { return side ? 80 - s : s; }

static int promotable(int t) { return t == FU || t == KY || t == KE || t == GI || t == KA || t == HI; }
static int promote(int t) { return t <= GI ? t + 8 : t == KA ? UM : RY; }
static int unpromote(int t) { return t >= TO && t <= NG ? t - 8 : t == UM ? KA : t == RY ? HI : t; }

/* Does a piece of type t (owned by the viewer "us", mover frame) at (r,c)
 * attack (tr,tc) given the board accessor? Steps + slides. */
typedef struct { const spos* p; int side; } view;
static inline uint8_t vat(const view* v, int r, int c) { return v->p->sq[fr(v->side, r * 9 + c)]; }
static inline int vown(const view* v, uint8_t pc) { return pc && SCOLOR(pc) == v->side; }

/* Is mover-frame square (r,c) attacked by the OPPONENT of v->side? */
static int attacked_by_opp(const view* v, int r, int c) {
    int opp = 1 - v->side;
    /* opponent moves "down" in our frame: an opponent piece at (r+dr', c+dc') attacks us where its
       own-frame offset is (-dr', -dc') rotated... easier: check every opponent piece's attacks. */
    for (int rr = 0; rr < 9; rr++)
        for (int cc = 0; cc < 9; cc++) {
            uint8_t pc = vat(v, rr, cc);
            if (!pc || SCOLOR(pc) != opp) continue;
            int t = STYPE(pc);
            /* opponent offsets are ours negated */
            int dr = r - rr, dc = c - cc;
            switch (t) {
                case FU: if (dr == 1 && dc == 0) return 1; break;
                case KE: if (dr == 2 && (dc == 1 || dc == -1)) return 1; break;
                case GI:
                    for (int k = 0; k < 5; k++) { if (-SILVER_D[k][0] == dr && -SILVER_D[k][1] == dc) return 1; }
                    break;
                case KI: case TO: case NY: case NK: case NG:
                    for (int k = 0; k < 6; k++) { if (-GOLD_D[k][0] == dr && -GOLD_D[k][1] == dc) return 1; }
                    break;
                case OU: if (dr >= -1 && dr <= 1 && dc >= -1 && dc <= 1 && (dr || dc)) return 1; break;
                default: break;
            }
            if (t == UM || t == RY) {
                if (dr >= -1 && dr <= 1 && dc >= -1 && dc <= 1 && (dr || dc)) return 1;
            }
            /* sliders: KY (opp forward = +row in our frame), KA/UM diagonals, HI/RY orthogonals */
            int slide_ok = 0, sr = 0, sc = 0;
            if (t == KY && dc == 0 && dr > 0) { slide_ok = 1; sr = 1; sc = 0; }
            if ((t == KA || t == UM) && dr != 0 && (dr == dc || dr == -dc)) { slide_ok = 1; sr = dr > 0 ? 1 : -1; sc = dc > 0 ? 1 : -1; }
            if ((t == HI || t == RY) && ((dr == 0) != (dc == 0))) { slide_ok = 1; sr = (dr > 0) - (dr < 0); sc = (dc > 0) - (dc < 0); }
            if (slide_ok) {
                int ir = rr + sr, ic = cc + sc, blocked = 0;
                while (ir != r || ic != c) {
                    if (vat(v, ir, ic)) { blocked = 1; break; }
                    ir += sr; ic += sc;
                }
                if (!blocked) return 1;
            }
        }
    return 0;
}

static int king_rc(const view* v, int* kr, int* kc) {
    for (int r = 0; r < 9; r++)
        for (int c = 0; c < 9; c++)
            if (vat(v, r, c) == SMK(v->side, OU)) { *kr = r; *kc = c; return 1; }
    return 0;
}

static int side_in_check(const spos* p, int side) {
    view v = {p, side};
    int kr, kc;
    if (!king_rc(&v, &kr, &kc)) return 0;
    return attacked_by_opp(&v, kr, kc);
}

/* make a move given in the mover's frame */
static void smake(spos* p, smove m) {
    int side = p->stm;
    int to = fr(side, m.to);
    if (m.drop) {
        int hi = m.drop - 1;
        p->hand[side][hi]--;
        static const uint8_t HT[7] = {FU, KY, KE, GI, KI, KA, HI};
        p->sq[to] = SMK(side, HT[hi]);
    } else {
        int from = fr(side, m.from);
        uint8_t pc = p->sq[from], cap = p->sq[to];
        if (cap) {
            int ct = unpromote(STYPE(cap));
            static const int8_t HI_OF[16] = {-1, 0, 1, 2, 3, 4, 5, 6, -1};
            p->hand[side][HI_OF[ct]]++;
        }
        p->sq[to] = m.promo ? SMK(side, promote(STYPE(pc))) : pc;
        p->sq[from] = E;
    }
    p->stm ^= 1;
}

static int gen_pseudo(const spos* p, smove* out) {
    int side = p->stm, n = 0;
    view v = {p, side};
    for (int r = 0; r < 9; r++)
        for (int c = 0; c < 9; c++) {
            uint8_t pc = vat(&v, r, c);
            if (!vown(&v, pc)) continue;
            int t = STYPE(pc), from = r * 9 + c;
            int8_t d[16][2]; int nd = 0, slides[8][2], ns = 0;
            switch (t) {
                case FU: d[nd][0] = -1; d[nd][1] = 0; nd++; break;
                case KY: slides[ns][0] = -1; slides[ns][1] = 0; ns++; break;
                case KE: d[nd][0] = -2; d[nd][1] = -1; nd++; d[nd][0] = -2; d[nd][1] = 1; nd++; break;
                case GI: for (int k = 0; k < 5; k++) { d[nd][0] = SILVER_D[k][0]; d[nd][1] = SILVER_D[k][1]; nd++; } break;
                case KI: case TO: case NY: case NK: case NG:
                    for (int k = 0; k < 6; k++) { d[nd][0] = GOLD_D[k][0]; d[nd][1] = GOLD_D[k][1]; nd++; } break;
                case OU: for (int k = 0; k < 8; k++) { d[nd][0] = KING_D[k][0]; d[nd][1] = KING_D[k][1]; nd++; } break;
                case KA: for (int k = 0; k < 4; k++) { slides[ns][0] = DIAG[k][0]; slides[ns][1] = DIAG[k][1]; ns++; } break;
                case HI: for (int k = 0; k < 4; k++) { slides[ns][0] = ORTH[k][0]; slides[ns][1] = ORTH[k][1]; ns++; } break;
                case UM: for (int k = 0; k < 4; k++) { slides[ns][0] = DIAG[k][0]; slides[ns][1] = DIAG[k][1]; ns++;
                                                        d[nd][0] = ORTH[k][0]; d[nd][1] = ORTH[k][1]; nd++; } break;
                case RY: for (int k = 0; k < 4; k++) { slides[ns][0] = ORTH[k][0]; slides[ns][1] = ORTH[k][1]; ns++;
                                                        d[nd][0] = DIAG[k][0]; d[nd][1] = DIAG[k][1]; nd++; } break;
            }
            int tos[40], ntos = 0;
            for (int k = 0; k < nd; k++) {
                int rr = r + d[k][0], cc = c + d[k][1];
                if (!son(rr, cc) || vown(&v, vat(&v, rr, cc))) continue;
                tos[ntos++] = rr * 9 + cc;
            }
            for (int k = 0; k < ns; k++) {
                int rr = r + slides[k][0], cc = c + slides[k][1];
                while (son(rr, cc)) {
                    uint8_t q = vat(&v, rr, cc);
                    if (vown(&v, q)) break;
                    tos[ntos++] = rr * 9 + cc;
                    if (q) break;
                    rr += slides[k][0]; cc += slides[k][1];
                }
            }
            for (int k = 0; k < ntos; k++) {
                int to = tos[k], trow = to / 9;
                int can_promo = promotable(t) && (r <= 2 || trow <= 2);
                int must = (t == FU || t == KY) ? trow == 0 : t == KE ? trow <= 1 : 0;
                if (can_promo) out[n++] = (smove){(int8_t)from, (uint8_t)to, 1, 0};
                if (!must) out[n++] = (smove){(int8_t)from, (uint8_t)to, 0, 0};
            }
        }
    /* drops */
    static const uint8_t HT[7] = {FU, KY, KE, GI, KI, KA, HI};
    for (int hi = 0; hi < 7; hi++) {
        if (!p->hand[side][hi]) continue;
        int t = HT[hi];
        for (int to = 0; to < 81; to++) {
            int r = to / 9, c = to % 9;
            if (vat(&v, r, c)) continue;
            if ((t == FU || t == KY) && r == 0) continue;
            if (t == KE && r <= 1) continue;
            if (t == FU) {
                int nifu = 0;
                for (int rr = 0; rr < 9; rr++) if (vat(&v, rr, c) == SMK(side, FU)) nifu = 1;
                if (nifu) continue;
            }
            out[n++] = (smove){-1, (uint8_t)to, 0, (uint8_t)(hi + 1)};
        }
    }
    return n;
}

static int gen_legal(const spos* p, smove* out);

/* legal = own king not attacked after the move; pawn drops that mate are illegal */
static int is_legal(const spos* p, smove m) {
    spos q = *p;
    smake(&q, m);
    if (side_in_check(&q, p->stm)) return 0;
    if (m.drop == 1 && side_in_check(&q, q.stm)) {   /* uchifuzume: pawn-drop check with no reply */
        smove buf[1024];
        if (gen_legal(&q, buf) == 0) return 0;
    }
    return 1;
}

static int gen_legal(const spos* p, smove* out) {
    smove tmp[1024];
    int n = gen_pseudo(p, tmp), k = 0;
    for (int i = 0; i < n; i++) if (is_legal(p, tmp[i])) out[k++] = tmp[i];
    return k;
}

/* action = dir * 81 + to (mover frame) */
static int action_of(smove m) {
    if (m.drop) return (20 + m.drop - 1) * 81 + m.to;
    int fr_ = m.from / 9, fc = m.from % 9, tr = m.to / 9, tc = m.to % 9;
    int dr = tr - fr_, dc = tc - fc, dir;
    if (dr == -2 && (dc == 1 || dc == -1)) dir = dc < 0 ? 8 : 9;   /* knight jump */
    else {
        int sr = (dr > 0) - (dr < 0), sc = (dc > 0) - (dc < 0);
        static const int DIRMAP[3][3] = {{1, 0, 2}, {3, -1, 4}, {6, 5, 7}};
        dir = DIRMAP[sr + 1][sc + 1];
    }
    return (dir + (m.promo ? 10 : 0)) * 81 + m.to;
}

static uint64_t pos_key(const spos* p) {
    uint64_t h = 0;
    for (int s = 0; s < 81; s++) if (p->sq[s]) h ^= orc_mix64(0x5306100000000000ULL + (uint64_t)p->sq[s] * 128 + (uint64_t)s);
    for (int c = 0; c < 2; c++)
        for (int i = 0; i < 7; i++)
            if (p->hand[c][i]) h ^= orc_mix64(0x5306200000000000ULL + (uint64_t)(c * 8 + i) * 32 + p->hand[c][i]);
    if (p->stm) h ^= orc_mix64(0x5306300000000000ULL);
    return h;
}

static const char* START_SFEN = "lnsgkgsnl/1r5b1/ppppppppp/9/9/9/PPPPPPPPP/1B5R1/LNSGKGSNL b - 1";

static int parse_sfen(const char* s, spos* p) {
    memset(p, 0, sizeof(*p));
    int r = 0, c = 0, prom = 0;
    const char* x = s;
    for (; *x && *x != ' '; x++) {
        if (*x == '/') { r++; c = 0; continue; }
        if (*x >= '1' && *x <= '9') { c += *x - '0'; continue; }
        if (*x == '+') { prom = 1; continue; }
        int color = (*x >= 'a') ? 1 : 0, t = 0;
        switch (*x | 32) { case 'p': t = FU; break; case 'l': t = KY; break; case 'n': t = KE; break; case 's': t = GI; break;
                           case 'g': t = KI; break; case 'b': t = KA; break; case 'r': t = HI; break; case 'k': t = OU; break;
                           default: return -1; }
        if (prom) t = promote(t);
        prom = 0;
        if (r > 8 || c > 8) return -1;
        p->sq[r * 9 + c++] = SMK(color, t);
    }
    if (*x) x++;
    p->stm = *x == 'w';
    while (*x && *x != ' ') x++;
    if (*x) x++;
    int cnt = 0;
    for (; *x && *x != ' '; x++) {
        if (*x == '-') break;
        if (*x >= '0' && *x <= '9') { cnt = cnt * 10 + (*x - '0'); continue; }
        int color = (*x >= 'a') ? 1 : 0, hi = -1;
        switch (*x | 32) { case 'p': hi = 0; break; case 'l': hi = 1; break; case 'n': hi = 2; break; case 's': hi = 3; break;
                           case 'g': hi = 4; break; case 'b': hi = 5; break; case 'r': hi = 6; break; default: return -1; }
        p->hand[color][hi] += (uint8_t)(cnt ? cnt : 1);
        cnt = 0;
    }
    return 0;
}

static void settle(orc_shogi* g, sg_env* e) {
    smove mv[1024];
    int n = gen_legal(&e->pos, mv);
    memset(e->mask, 0, SG_A);
    for (int i = 0; i < n; i++) e->mask[action_of(mv[i])] = 1;
    uint64_t key = pos_key(&e->pos);
    int reps = 0;
    for (int j = 0; j < e->step_count; j++) reps += e->hist[j] == key;
    e->hist[e->step_count] = key;
    e->rep = (uint8_t)(reps > 3 ? 3 : reps);
    e->in_check = (uint8_t)side_in_check(&e->pos, e->pos.stm);
    e->terminal = 0;
    e->role_rewards[0] = e->role_rewards[1] = 0.0f;
    if (n == 0) {   /* no legal move: the side to move loses (no stalemate in shogi) */
        e->terminal = 1;
        e->role_rewards[e->pos.stm] = -1.0f;
        e->role_rewards[1 - e->pos.stm] = 1.0f;
    } else if (reps >= 3) {   /* four-fold repetition: draw */
        e->terminal = 1;
    }
    if (e->terminal) memset(e->mask, 0, SG_A);
}

static void env_init(orc_shogi* g, sg_env* e, uint64_t key) {
    uint64_t c = orc_child(key, 0) % 2;
    e->p2r[0] = (int8_t)c; e->p2r[1] = (int8_t)(1 - c);
    parse_sfen(START_SFEN, &e->pos);
    e->step_count = 0; e->truncated = 0;
    settle(g, e);
}

static void env_apply(orc_shogi* g, sg_env* e, int action) {
    smove mv[1024];
    int n = gen_legal(&e->pos, mv);
    for (int i = 0; i < n; i++)
        if (action_of(mv[i]) == action) { smake(&e->pos, mv[i]); break; }
    e->step_count += 1;
    settle(g, e);
}

orc_shogi* orc_shogi_new(int64_t n, int max_steps) {
    orc_shogi* g = (orc_shogi*)calloc(1, sizeof(orc_shogi));
    g->n = n; g->max_steps = max_steps;
    g->env = (sg_env*)calloc((size_t)n, sizeof(sg_env));
    for (int64_t i = 0; i < n; i++) g->env[i].hist = (uint64_t*)calloc((size_t)max_steps + 2, sizeof(uint64_t));
    return g;
}

void orc_shogi_free(orc_shogi* g) {
    if (!g) return;
    for (int64_t i = 0; i < g->n; i++) free(g->env[i].hist);
    free(g->env); free(g);
}

void orc_shogi_init(orc_shogi* g, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) env_init(g, &g->env[i], orc_slot_key(slot_keys, key_state, slot0, i));
}

int64_t orc_shogi_step(orc_shogi* g, const int64_t* actions, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    for (int64_t i = 0; i < g->n; i++) {
        sg_env* e = &g->env[i];
        if (e->terminal || e->truncated) continue;
        int64_t a = actions[i];
        if (a < 0 || a >= SG_A || !e->mask[a]) return i;
    }
    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < g->n; i++) {
        sg_env* e = &g->env[i];
        uint64_t k = orc_slot_key(slot_keys, key_state, slot0, i);
        if (e->terminal || e->truncated) { env_init(g, e, k); continue; }
        env_apply(g, e, (int)actions[i]);
        e->truncated = (uint8_t)(!e->terminal && e->step_count >= g->max_steps);
        if (e->truncated) memset(e->mask, 0, SG_A);
    }
    return -1;
}

/* Observation (dlshogi-style) for `role`, mover frame:
 *   0-13 own pieces by type, 14-27 squares attacked by own pieces of each type,
 *   28-30 attacked by >= 1/2/3 own pieces, 31-61 the same for the opponent,
 *   62-89 own hand (FU 8, KY 4, KE 4, GI 4, KI 4, KA 2, HI 2 threshold planes),
 *   90-117 opponent hand, 118 own king in check. */
static int attacks_of(const view* v, int r, int c, int* out) {   /* squares attacked by the piece at (r,c) */
    uint8_t pc = vat(v, r, c);
    int t = STYPE(pc), owner = SCOLOR(pc), n = 0;
    int sgn = owner == v->side ? 1 : -1;   /* opponent pieces move downward in our frame */
    int8_t d[16][2]; int nd = 0; int8_t sl[8][2]; int ns = 0;
    switch (t) {
        case FU: d[nd][0] = -1; d[nd][1] = 0; nd++; break;
        case KY: sl[ns][0] = -1; sl[ns][1] = 0; ns++; break;
        case KE: d[nd][0] = -2; d[nd][1] = -1; nd++; d[nd][0] = -2; d[nd][1] = 1; nd++; break;
        case GI: for (int k = 0; k < 5; k++) { d[nd][0] = SILVER_D[k][0]; d[nd][1] = SILVER_D[k][1]; nd++; } break;
        case KI: case TO: case NY: case NK: case NG:
            for (int k = 0; k < 6; k++) { d[nd][0] = GOLD_D[k][0]; d[nd][1] = GOLD_D[k][1]; nd++; } break;
        case OU: for (int k = 0; k < 8; k++) { d[nd][0] = KING_D[k][0]; d[nd][1] = KING_D[k][1]; nd++; } break;
        case KA: for (int k = 0; k < 4; k++) { sl[ns][0] = DIAG[k][0]; sl[ns][1] = DIAG[k][1]; ns++; } break;
        case HI: for (int k = 0; k < 4; k++) { sl[ns][0] = ORTH[k][0]; sl[ns][1] = ORTH[k][1]; ns++; } break;
        case UM: for (int k = 0; k < 4; k++) { sl[ns][0] = DIAG[k][0]; sl[ns][1] = DIAG[k][1]; ns++;
                                                d[nd][0] = ORTH[k][0]; d[nd][1] = ORTH[k][1]; nd++; } break;
        case RY: for (int k = 0; k < 4; k++) { sl[ns][0] = ORTH[k][0]; sl[ns][1] = ORTH[k][1]; ns++;
                                                d[nd][0] = DIAG[k][0]; d[nd][1] = DIAG[k][1]; nd++; } break;
    }
    for (int k = 0; k < nd; k++) {
        int rr = r + sgn * d[k][0], cc = c + sgn * d[k][1];
        if (son(rr, cc)) out[n++] = rr * 9 + cc;
    }
    for (int k = 0; k < ns; k++) {
        int rr = r + sgn * sl[k][0], cc = c + sgn * sl[k][1];
        while (son(rr, cc)) {
            out[n++] = rr * 9 + cc;
            if (vat(v, rr, cc)) break;
            rr += sgn * sl[k][0]; cc += sgn * sl[k][1];
        }
    }
    return n;
}

void orc_shogi_observe(const orc_shogi* g, int64_t i, int role, float* obs) {
    const sg_env* e = &g->env[i];
    view v = {&e->pos, role};
    memset(obs, 0, sizeof(float) * SG_OBS);
    int cnt[2][81];
    memset(cnt, 0, sizeof(cnt));
    for (int r = 0; r < 9; r++)
        for (int c = 0; c < 9; c++) {
            uint8_t pc = vat(&v, r, c);
            if (!pc) continue;
            int who = SCOLOR(pc) == role ? 0 : 1, t = STYPE(pc);
            obs[(r * 9 + c) * 119 + 31 * who + t - 1] = 1.0f;
            int tg[64];
            int n = attacks_of(&v, r, c, tg);
            for (int k = 0; k < n; k++) {
                obs[tg[k] * 119 + 31 * who + 14 + t - 1] = 1.0f;
                cnt[who][tg[k]]++;
            }
        }
    static const int HCAP[7] = {8, 4, 4, 4, 4, 2, 2};
    static const int HOFF[7] = {0, 8, 12, 16, 20, 24, 26};
    for (int s = 0; s < 81; s++) {
        float* o = obs + s * 119;
        for (int who = 0; who < 2; who++) {
            for (int k = 0; k < 3; k++) if (cnt[who][s] > k) o[31 * who + 28 + k] = 1.0f;
            int owner = who == 0 ? role : 1 - role;
            for (int hi = 0; hi < 7; hi++)
                for (int k = 0; k < HCAP[hi]; k++)
                    if (e->pos.hand[owner][hi] > k) o[62 + 28 * who + HOFF[hi] + k] = 1.0f;
        }
        o[118] = side_in_check(&e->pos, role) ? 1.0f : 0.0f;
    }
}

void orc_shogi_columns(const orc_shogi* g, float* obs, uint8_t* mask, float* rewards, uint8_t* term,
                       uint8_t* trunc, int32_t* cur, int32_t* step_count, int8_t* p2r) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) {
        const sg_env* e = &g->env[i];
        if (mask) memcpy(mask + i * SG_A, e->mask, SG_A);
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
        if (obs) orc_shogi_observe(g, i, e->pos.stm, obs + (size_t)i * SG_OBS);
    }
}

/* encode: board[81] + hands[2][7] + stm + repetition count */
int orc_shogi_encode(const orc_shogi* g, int64_t i, uint8_t* buf) {
    const sg_env* e = &g->env[i];
    memcpy(buf, e->pos.sq, 81);
    memcpy(buf + 81, e->pos.hand, 14);
    buf[95] = e->pos.stm;
    buf[96] = e->rep;
    return 97;
}

static uint64_t sperft(const spos* p, int depth) {
    smove mv[1024];
    int n = gen_legal(p, mv);
    if (depth == 1) return (uint64_t)n;
    uint64_t total = 0;
    for (int i = 0; i < n; i++) {
        spos q = *p;
        smake(&q, mv[i]);
        total += sperft(&q, depth - 1);
    }
    return total;
}

uint64_t orc_shogi_perft(const char* sfen, int depth) {
    spos p;
    if (parse_sfen(sfen ? sfen : START_SFEN, &p) != 0) return 0;
    return depth <= 0 ? 1 : sperft(&p, depth);
}

int orc_shogi_set_sfen(orc_shogi* g, int64_t i, const char* sfen) {
    sg_env* e = &g->env[i];
    if (parse_sfen(sfen, &e->pos) != 0) return -1;
    e->step_count = 0; e->terminal = 0; e->truncated = 0;
    settle(g, e);
    return 0;
}
