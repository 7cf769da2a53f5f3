/* ORACLE (test infrastructure only) -- Go, CPU restatement of the reference.
 *
 * Follows reference pkg/src/boardbatch/games/go.py function by function:
 *   zobrist            go.py:20-25     neighbour table  go.py:28-42
 *   analyse (DFS)      go.py:45-80     Core.encode      go.py:103-111
 *   legal_mask         go.py:121-174   score_rewards    go.py:176-210
 *   init_core          go.py:212-217   apply            go.py:219-262
 *   observe            go.py:264-273   _flood_group     go.py:293-309
 * and the env-core wrapping of pkg/src/boardbatch/core.py:
 *   init  core.py:223-229, step core.py:232-243, _make_state core.py:192-220,
 *   batch_step auto-reset core.py:353-386.
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load this code. It is the checker, never the product.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "orc_rng.h"

#define GO_MAXN 25
#define GO_MAXC (GO_MAXN * GO_MAXN)
#define GO_HIST 8

typedef struct {
    uint64_t* slot;  /* open addressing, 0 slot value marks empty -> track zero separately */
    uint32_t cap;    /* power of two */
    int32_t count;   /* len(history) */
    uint8_t has_zero;
} hset;

typedef struct {
    uint8_t board[GO_MAXC];
    uint8_t role_to_move, pass_count, terminal, truncated;
    float role_rewards[2];
    uint64_t hash, hist_xor;
    hset history;
    uint8_t bh[GO_HIST][GO_MAXC];
    int nbh;
    /* analysis cache (Core.an) */
    int16_t group_of[GO_MAXC];
    int16_t libs[GO_MAXC];
    uint64_t gxor[GO_MAXC];
    int16_t ghead[GO_MAXC], gnext[GO_MAXC];
    int ngroups;
    uint8_t mask[GO_MAXC + 1]; /* core.mask as bytes */
    int32_t step_count;
    int8_t p2r[2];
} go_env;

typedef struct {
    int N, cells, A, max_steps, self_capture;
    double komi;
    int64_t n;
    uint64_t zob[2][GO_MAXC];
    int16_t nbr[GO_MAXC][4];
    uint8_t nnbr[GO_MAXC];
    go_env* env;
    go_env* scratch; /* used for the all-or-nothing illegal check */
} orc_go;

/* ---------------- history set ---------------- */
static void hs_clear(hset* s) {
    memset(s->slot, 0, sizeof(uint64_t) * s->cap);
    s->count = 0;
    s->has_zero = 0;
}
static int hs_has(const hset* s, uint64_t h) {
    if (h == 0) return s->has_zero;
    uint32_t m = s->cap - 1, i = (uint32_t)(h ^ (h >> 32)) & m;
    while (s->slot[i]) {
        if (s->slot[i] == h) return 1;
        i = (i + 1) & m;
    }
    return 0;
}
static void hs_add(hset* s, uint64_t h) {
    if (hs_has(s, h)) return;
    s->count++;
    if (h == 0) { s->has_zero = 1; return; }
    uint32_t m = s->cap - 1, i = (uint32_t)(h ^ (h >> 32)) & m;
    while (s->slot[i]) i = (i + 1) & m;
    s->slot[i] = h;
}

/* ---------------- analysis: go.py:45-80 ---------------- */
static void analyse(const orc_go* g, go_env* e) {
    int cells = g->cells;
    int16_t stamp[GO_MAXC];
    int16_t stack[GO_MAXC];
    for (int i = 0; i < cells; i++) { e->group_of[i] = -1; stamp[i] = -1; }
    int ng = 0;
    for (int i = 0; i < cells; i++) {
        int color = e->board[i];
        if (color == 0 || e->group_of[i] >= 0) continue;
        int gid = ng++;
        const uint64_t* zc = g->zob[color - 1];
        int sp = 0;
        stack[sp++] = (int16_t)i;
        e->group_of[i] = (int16_t)gid;
        int libc = 0;
        uint64_t x = 0;
        int16_t head = -1;
        while (sp) {
            int p = stack[--sp];
            e->gnext[p] = head; head = (int16_t)p;  /* stone list */
            x ^= zc[p];
            for (int k = 0; k < g->nnbr[p]; k++) {
                int q = g->nbr[p][k];
                int v = e->board[q];
                if (v == 0) {
                    if (stamp[q] != gid) { stamp[q] = (int16_t)gid; libc++; }
                } else if (v == color && e->group_of[q] < 0) {
                    e->group_of[q] = (int16_t)gid;
                    stack[sp++] = (int16_t)q;
                }
            }
        }
        e->libs[gid] = (int16_t)libc;
        e->ghead[gid] = head;
        e->gxor[gid] = x;
    }
    e->ngroups = ng;
}

/* ---------------- legal mask: go.py:121-174 ---------------- */
static void legal_mask(const orc_go* g, go_env* e, int color, uint64_t h) {
    int cells = g->cells;
    const uint64_t* zc = g->zob[color - 1];
    memset(e->mask, 0, (size_t)g->A);
    e->mask[cells] = 1; /* pass always legal */
    for (int p = 0; p < cells; p++) {
        if (e->board[p]) continue;
        int empty_nbr = 0, helped = 0, ncaps = 0;
        int caps[4];
        for (int k = 0; k < g->nnbr[p]; k++) {
            int q = g->nbr[p][k];
            int v = e->board[q];
            if (v == 0) {
                empty_nbr = 1;
            } else if (v == color) {
                if (e->libs[e->group_of[q]] >= 2) helped = 1;
            } else {
                int gg = e->group_of[q];
                if (e->libs[gg] == 1) {
                    int dup = 0;
                    for (int j = 0; j < ncaps; j++) dup |= caps[j] == gg;
                    if (!dup) caps[ncaps++] = gg;
                }
            }
        }
        if (ncaps) {
            uint64_t h2 = h ^ zc[p];
            for (int j = 0; j < ncaps; j++) h2 ^= e->gxor[caps[j]];
            if (!hs_has(&e->history, h2)) e->mask[p] = 1;
        } else if (empty_nbr || helped) {
            if (!hs_has(&e->history, h ^ zc[p])) e->mask[p] = 1;
        } else if (g->self_capture) {
            uint64_t h2 = h;
            int own[4], nown = 0;
            for (int k = 0; k < g->nnbr[p]; k++) {
                int q = g->nbr[p][k];
                if (e->board[q] == color) {
                    int gg = e->group_of[q], dup = 0;
                    for (int j = 0; j < nown; j++) dup |= own[j] == gg;
                    if (!dup) own[nown++] = gg;
                }
            }
            for (int j = 0; j < nown; j++) h2 ^= e->gxor[own[j]];
            if (!hs_has(&e->history, h2)) e->mask[p] = 1;
        }
    }
}

/* ---------------- Tromp-Taylor score: go.py:176-210 ---------------- */
static void score_rewards(const orc_go* g, const uint8_t* board, float* rr) {
    double black = 0, white = 0;
    int cells = g->cells;
    for (int i = 0; i < cells; i++) {
        if (board[i] == 1) black += 1;
        else if (board[i] == 2) white += 1;
    }
    uint8_t seen[GO_MAXC];
    int16_t stack[GO_MAXC];
    memset(seen, 0, (size_t)cells);
    for (int i = 0; i < cells; i++) {
        if (board[i] != 0 || seen[i]) continue;
        seen[i] = 1;
        int sp = 0, region = 1, borders = 0;
        stack[sp++] = (int16_t)i;
        while (sp) {
            int p = stack[--sp];
            for (int k = 0; k < g->nnbr[p]; k++) {
                int q = g->nbr[p][k];
                int v = board[q];
                if (v == 0) {
                    if (!seen[q]) { seen[q] = 1; region++; stack[sp++] = (int16_t)q; }
                } else {
                    borders |= v;
                }
            }
        }
        if (borders == 1) black += region;
        else if (borders == 2) white += region;
    }
    white += g->komi;
    if (black > white) { rr[0] = 1.0f; rr[1] = -1.0f; }
    else if (white > black) { rr[0] = -1.0f; rr[1] = 1.0f; }
    else { rr[0] = 0.0f; rr[1] = 0.0f; }
}

static void push_hist(const orc_go* g, go_env* e) {
    /* boards_hist = (board,) + boards_hist[:7]  (go.py:224, 260) */
    int keep = e->nbh < GO_HIST ? e->nbh : GO_HIST - 1;
    memmove(e->bh[1], e->bh[0], (size_t)keep * GO_MAXC);
    memcpy(e->bh[0], e->board, (size_t)g->cells);
    e->nbh = keep + 1;
}

/* init_core (go.py:212-217) + core.init (core.py:223-229) */
static void env_init(const orc_go* g, go_env* e, uint64_t key) {
    uint64_t c = orc_child(key, 0) % 2;
    e->p2r[0] = (int8_t)c;
    e->p2r[1] = (int8_t)(1 - c);
    memset(e->board, 0, (size_t)g->cells);
    e->role_to_move = 0; e->pass_count = 0; e->terminal = 0; e->truncated = 0;
    e->role_rewards[0] = e->role_rewards[1] = 0.0f;
    e->hash = 0; e->hist_xor = 0;
    hs_clear(&e->history);
    hs_add(&e->history, 0);
    memcpy(e->bh[0], e->board, (size_t)g->cells);
    e->nbh = 1;
    analyse(g, e);
    legal_mask(g, e, 1, 0);
    e->step_count = 0;
}

/* _flood_group (go.py:293-309) */
static int flood_group(const orc_go* g, const uint8_t* board, int start, int16_t* group, int* has_lib) {
    int color = board[start];
    uint8_t member[GO_MAXC];
    memset(member, 0, (size_t)g->cells);
    int n = 0, sp = 0;
    int16_t stack[GO_MAXC];
    group[n++] = (int16_t)start; member[start] = 1; stack[sp++] = (int16_t)start;
    *has_lib = 0;
    while (sp) {
        int p = stack[--sp];
        for (int k = 0; k < g->nnbr[p]; k++) {
            int q = g->nbr[p][k];
            int v = board[q];
            if (v == 0) *has_lib = 1;
            else if (v == color && !member[q]) { member[q] = 1; group[n++] = (int16_t)q; stack[sp++] = (int16_t)q; }
        }
    }
    return n;
}

/* apply (go.py:219-262) + step's _make_state (core.py:243) */
static void env_apply(const orc_go* g, go_env* e, int action) {
    int mover = e->role_to_move, color = mover + 1;
    int cells = g->cells;
    e->step_count += 1;
    if (action == cells) {
        e->pass_count += 1;
        push_hist(g, e);
        e->role_to_move = (uint8_t)(1 - mover);
        if (e->pass_count == 2) {
            e->terminal = 1;
            score_rewards(g, e->board, e->role_rewards);
            memset(e->mask, 0, (size_t)g->A);
            return;
        }
        e->role_rewards[0] = e->role_rewards[1] = 0.0f;
        legal_mask(g, e, 3 - color, e->hash);
        return;
    }
    const uint64_t* zc = g->zob[color - 1];
    int enemy = 3 - color;
    uint64_t h2 = e->hash ^ zc[action];
    int captured_any = 0;
    int seen[4], nseen = 0;
    for (int k = 0; k < g->nnbr[action]; k++) {
        int q = g->nbr[action][k];
        if (e->board[q] == enemy) {
            int gg = e->group_of[q], dup = 0;
            for (int j = 0; j < nseen; j++) dup |= seen[j] == gg;
            if (e->libs[gg] == 1 && !dup) {
                seen[nseen++] = gg;
                captured_any = 1;
                h2 ^= e->gxor[gg];
                for (int s = e->ghead[gg]; s >= 0; s = e->gnext[s]) e->board[s] = 0;
            }
        }
    }
    e->board[action] = (uint8_t)color;
    if (g->self_capture && !captured_any) {
        int16_t grp[GO_MAXC];
        int has_lib;
        int ngs = flood_group(g, e->board, action, grp, &has_lib);
        if (!has_lib) {
            for (int j = 0; j < ngs; j++) { e->board[grp[j]] = 0; h2 ^= zc[grp[j]]; }
        }
    }
    hs_add(&e->history, h2);
    analyse(g, e);
    legal_mask(g, e, enemy, h2);
    push_hist(g, e);
    e->role_to_move = (uint8_t)(1 - mover);
    e->pass_count = 0;
    e->hash = h2;
    e->hist_xor ^= h2;
    e->role_rewards[0] = e->role_rewards[1] = 0.0f;
}

/* ---------------- public API ---------------- */
orc_go* orc_go_new(int size, double komi, int self_capture, int64_t n, int max_steps) {
    if (size < 2 || size > GO_MAXN || n < 1) return NULL;
    orc_go* g = (orc_go*)calloc(1, sizeof(orc_go));
    g->N = size; g->cells = size * size; g->A = g->cells + 1;
    g->komi = komi; g->self_capture = self_capture; g->n = n; g->max_steps = max_steps;
    uint64_t base = 0x60D00D60C0FFEE00ULL + (uint64_t)size;   /* go.py:22 */
    for (int i = 0; i < g->cells; i++) {
        g->zob[0][i] = orc_mix64(base + 2ULL * (uint64_t)i);
        g->zob[1][i] = orc_mix64(base + 2ULL * (uint64_t)i + 1);
    }
    for (int r = 0; r < size; r++)
        for (int c = 0; c < size; c++) {   /* order matches go.py:32-40 */
            int i = r * size + c, k = 0;
            if (r > 0) g->nbr[i][k++] = (int16_t)((r - 1) * size + c);
            if (r < size - 1) g->nbr[i][k++] = (int16_t)((r + 1) * size + c);
            if (c > 0) g->nbr[i][k++] = (int16_t)(r * size + c - 1);
            if (c < size - 1) g->nbr[i][k++] = (int16_t)(r * size + c + 1);
            g->nnbr[i] = (uint8_t)k;
        }
    g->env = (go_env*)calloc((size_t)n, sizeof(go_env));
    g->scratch = NULL;
    uint32_t cap = 64;
    while (cap < 2u * (uint32_t)(max_steps + 2)) cap <<= 1;
    for (int64_t i = 0; i < n; i++) {
        g->env[i].history.cap = cap;
        g->env[i].history.slot = (uint64_t*)calloc(cap, sizeof(uint64_t));
    }
    return g;
}

void orc_go_free(orc_go* g) {
    if (!g) return;
    for (int64_t i = 0; i < g->n; i++) free(g->env[i].history.slot);
    free(g->env);
    free(g);
}

/* batch_init (core.py:340-350): slot i uses key.child(slot0 + i). */
void orc_go_init(orc_go* g, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < g->n; i++) env_init(g, &g->env[i], orc_slot_key(slot_keys, key_state, slot0, i));
}

/* batch_step (core.py:353-386). Returns -1, or the lowest offending live
 * slot with every state left unchanged (tictactoe.py:111-121 semantics). */
int64_t orc_go_step(orc_go* g, const int64_t* actions, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    for (int64_t i = 0; i < g->n; i++) {
        go_env* e = &g->env[i];
        if (e->terminal || e->truncated) continue;
        int64_t a = actions[i];
        if (a < 0 || a >= g->A || !e->mask[a]) return i;
    }
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < g->n; i++) {
        go_env* e = &g->env[i];
        uint64_t k = orc_slot_key(slot_keys, key_state, slot0, i);
        if (e->terminal || e->truncated) { env_init(g, e, k); continue; }
        env_apply(g, e, (int)actions[i]);
        e->truncated = (uint8_t)(!e->terminal && e->step_count >= g->max_steps);  /* core.py:196 */
    }
    return -1;
}

/* observe (go.py:264-273) for one slot and role. */
void orc_go_observe(const orc_go* g, int64_t i, int role, float* out) {
    const go_env* e = &g->env[i];
    int N = g->N, cells = g->cells, P = 2 * GO_HIST + 1;
    int mine = role + 1, theirs = 2 - role;
    memset(out, 0, sizeof(float) * (size_t)cells * (size_t)P);
    for (int c = 0; c < cells; c++) {
        for (int t = 0; t < e->nbh; t++) {
            out[c * P + 2 * t] = e->bh[t][c] == mine ? 1.0f : 0.0f;
            out[c * P + 2 * t + 1] = e->bh[t][c] == theirs ? 1.0f : 0.0f;
        }
        out[c * P + 2 * GO_HIST] = (float)role;
    }
    (void)N;
}

/* Public columns, _make_state (core.py:192-220); obs = batch_outputs
 * (bench.py:86-97): observe(s, s.current_player). Any pointer may be NULL. */
void orc_go_columns(const orc_go* g, float* obs, uint8_t* mask, float* rewards, uint8_t* term,
                    uint8_t* trunc, int32_t* cur, int32_t* step_count, int8_t* p2r) {
    int A = g->A;
    size_t osz = (size_t)g->cells * (2 * GO_HIST + 1);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) {
        const go_env* e = &g->env[i];
        int fin = e->terminal || e->truncated;
        if (mask) {
            if (fin) memset(mask + i * A, 0, (size_t)A);
            else memcpy(mask + i * A, e->mask, (size_t)A);
        }
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
        if (cur) cur[i] = e->p2r[0] == e->role_to_move ? 0 : 1;
        if (step_count) step_count[i] = e->step_count;
        if (p2r) { p2r[2 * i] = e->p2r[0]; p2r[2 * i + 1] = e->p2r[1]; }
        if (obs) orc_go_observe(g, i, e->role_to_move, obs + (size_t)i * osz);
    }
}

/* Core.encode (go.py:103-111). Returns the byte length. */
int orc_go_encode(const orc_go* g, int64_t i, uint8_t* buf) {
    const go_env* e = &g->env[i];
    int cells = g->cells, o = 0;
    memcpy(buf, e->board, (size_t)cells); o += cells;
    buf[o++] = e->role_to_move;
    buf[o++] = e->pass_count;
    for (int k = 0; k < 8; k++) buf[o++] = (uint8_t)(e->hash >> (8 * k));
    for (int k = 0; k < 8; k++) buf[o++] = (uint8_t)(e->hist_xor >> (8 * k));
    buf[o++] = (uint8_t)(e->history.count & 0xFF);
    buf[o++] = (uint8_t)((e->history.count >> 8) & 0xFF);
    for (int t = 0; t < e->nbh; t++) { memcpy(buf + o, e->bh[t], (size_t)cells); o += cells; }
    return o;
}

/* Scalar internals used by tests (role_to_move, terminal, hash, ...). */
void orc_go_scalars(const orc_go* g, int64_t i, int64_t* out6) {
    const go_env* e = &g->env[i];
    out6[0] = e->role_to_move; out6[1] = e->pass_count; out6[2] = e->terminal;
    out6[3] = (int64_t)e->hash; out6[4] = (int64_t)e->hist_xor; out6[5] = e->history.count;
}

/* Test hook: overwrite one slot's board/role and re-derive the analysis and mask. */
void orc_go_set_board(orc_go* g, int64_t i, const uint8_t* board, int role) {
    go_env* e = &g->env[i];
    memcpy(e->board, board, (size_t)g->cells);
    e->role_to_move = (uint8_t)role;
    analyse(g, e);
    legal_mask(g, e, role + 1, e->hash);
}
