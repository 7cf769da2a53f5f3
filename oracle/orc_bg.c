/* ORACLE (test infrastructure only) -- backgammon, CPU restatement.
 *
 * Follows reference pkg/src/boardbatch/games/backgammon.py:
 *   _abs_point :22-24, _signed :27-29, _legal_mask :62-95, Core.encode :113-119,
 *   _START_POINTS :122, _roll :125-130, _init_core :133-134, _final :137-147,
 *   _apply :150-193, _observe :196-206; and env-core core.py:192-243,353-386.
 * Only tests/, __graft_entry__.smoke() and bench.py may load this code.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include "orc_rng.h"

#define BG_A 156

typedef struct {
    int8_t points[24];
    uint8_t bar[2], off[2];
    uint8_t role_to_move, terminal, truncated;
    uint8_t dice[2];
    uint8_t rem[4];
    uint8_t nrem;
    float role_rewards[2];
    uint8_t mask[BG_A];
    int32_t step_count;
    int8_t p2r[2];
} bg_env;

typedef struct {
    int64_t n;
    int max_steps;
    bg_env* env;
} orc_bg;

static const int8_t START_POINTS[24] = {2, 0, 0, 0, 0, -5, 0, -3, 0, 0, 0, 5, -5, 0, 0, 0, 3, 0, 5, 0, 0, 0, 0, -2};

static inline int abs_point(int role, int pip) { return role == 0 ? 24 - pip : pip - 1; }
static inline int signed_at(const int8_t* pts, int role, int a) { return role == 0 ? pts[a] : -pts[a]; }

/* _legal_mask (backgammon.py:62-95) */
static void legal_mask(bg_env* e) {
    int role = e->role_to_move, sign = role == 0 ? 1 : -1;
    memset(e->mask, 0, BG_A);
    int any = 0;
    int dset[7] = {0};
    for (int j = 0; j < e->nrem; j++) dset[e->rem[j]] = 1;
    if (e->bar[role] > 0) {
        for (int die = 1; die <= 6; die++) {
            if (!dset[die]) continue;
            int dest = role == 0 ? 24 - (25 - die) : (25 - die) - 1;
            if (e->points[dest] * sign >= -1) { e->mask[6 + die - 1] = 1; any = 1; }
        }
        if (!any) e->mask[0] = 1;
        return;
    }
    int rear = 0;
    for (int a = 0; a < 24; a++) {
        if (e->points[a] * sign > 0) {
            int pip = role == 0 ? 24 - a : a + 1;
            if (pip > rear) rear = pip;
        }
    }
    int can_bear_off = rear <= 6;
    for (int die = 1; die <= 6; die++) {
        if (!dset[die]) continue;
        int bit = die - 1;
        for (int pip = 1; pip <= 24; pip++) {
            int src = role == 0 ? 24 - pip : pip - 1;
            if (e->points[src] * sign < 1) continue;
            int target = pip - die;
            if (target >= 1) {
                int dest = role == 0 ? 24 - target : target - 1;
                if (e->points[dest] * sign >= -1) { e->mask[(pip + 1) * 6 + bit] = 1; any = 1; }
            } else if (can_bear_off && (die == pip || pip == rear)) {
                e->mask[(pip + 1) * 6 + bit] = 1; any = 1;
            }
        }
    }
    if (!any) e->mask[0] = 1;
}

/* _roll (backgammon.py:125-130) */
static void roll(bg_env* e, int role, uint64_t key) {
    int d1 = (int)(orc_child(key, 0) % 6) + 1;
    int d2 = (int)(orc_child(key, 1) % 6) + 1;
    e->role_to_move = (uint8_t)role;
    e->dice[0] = (uint8_t)d1; e->dice[1] = (uint8_t)d2;
    if (d1 == d2) { e->nrem = 4; for (int j = 0; j < 4; j++) e->rem[j] = (uint8_t)d1; }
    else { e->nrem = 2; e->rem[0] = (uint8_t)d1; e->rem[1] = (uint8_t)d2; e->rem[2] = e->rem[3] = 0; }
    e->terminal = 0;
    e->role_rewards[0] = e->role_rewards[1] = 0.0f;
    legal_mask(e);
}

/* _final (backgammon.py:137-147) */
static void final_(bg_env* e, int winner) {
    int loser = 1 - winner;
    float value = 1.0f;
    if (e->off[loser] == 0) {
        value = 2.0f;
        int in_home = 0;
        int lo = winner == 0 ? 18 : 0;
        for (int a = lo; a < lo + 6; a++) in_home |= signed_at(e->points, loser, a) > 0;
        if (e->bar[loser] > 0 || in_home) value = 3.0f;
    }
    if (winner == 0) { e->role_rewards[0] = value; e->role_rewards[1] = -value; }
    else { e->role_rewards[0] = -value; e->role_rewards[1] = value; }
    e->role_to_move = (uint8_t)loser;
    e->dice[0] = e->dice[1] = 0;
    e->nrem = 0; memset(e->rem, 0, 4);
    e->terminal = 1;
    memset(e->mask, 0, BG_A);
}

/* init (core.py:223-229) with _init_core (backgammon.py:133-134) */
static void env_init(bg_env* e, uint64_t key) {
    uint64_t c = orc_child(key, 0) % 2;
    e->p2r[0] = (int8_t)c; e->p2r[1] = (int8_t)(1 - c);
    memcpy(e->points, START_POINTS, 24);
    e->bar[0] = e->bar[1] = 0; e->off[0] = e->off[1] = 0;
    e->truncated = 0;
    e->step_count = 0;
    roll(e, 0, orc_child(key, 1));
}

/* _apply (backgammon.py:150-193) */
static void env_apply(bg_env* e, int action, uint64_t key) {
    int role = e->role_to_move;
    int src = action / 6, die = action % 6 + 1;
    e->step_count += 1;
    if (src == 0) { roll(e, 1 - role, key); return; }
    int delta = role == 0 ? 1 : -1;
    int target;
    if (src == 1) { e->bar[role] -= 1; target = 25 - die; }
    else { int pip = src - 1; e->points[abs_point(role, pip)] -= (int8_t)delta; target = pip - die; }
    if (src != 1 && target < 1) {
        e->off[role] += 1;
    } else {
        int a = abs_point(role, target);
        if (signed_at(e->points, role, a) == -1) { e->points[a] = (int8_t)delta; e->bar[1 - role] += 1; }
        else e->points[a] += (int8_t)delta;
    }
    if (e->off[role] == 15) { final_(e, role); return; }
    /* remaining.remove(die): drop the first occurrence, keep order */
    int j = 0;
    while (j < e->nrem && e->rem[j] != die) j++;
    for (; j + 1 < e->nrem; j++) e->rem[j] = e->rem[j + 1];
    if (e->nrem > 0) { e->nrem -= 1; e->rem[e->nrem & 3] = 0; }
    if (e->nrem == 0) { roll(e, 1 - role, key); return; }
    e->role_rewards[0] = e->role_rewards[1] = 0.0f;
    legal_mask(e);
}

orc_bg* orc_bg_new(int64_t n, int max_steps) {
    if (n < 1) return NULL;
    orc_bg* g = (orc_bg*)calloc(1, sizeof(orc_bg));
    g->n = n; g->max_steps = max_steps;
    g->env = (bg_env*)calloc((size_t)n, sizeof(bg_env));
    return g;
}

void orc_bg_free(orc_bg* g) {
    if (!g) return;
    free(g->env);
    free(g);
}

void orc_bg_init(orc_bg* g, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) env_init(&g->env[i], orc_slot_key(slot_keys, key_state, slot0, i));
}

int64_t orc_bg_step(orc_bg* g, const int64_t* actions, uint64_t key_state, int64_t slot0, const uint64_t* slot_keys) {
    for (int64_t i = 0; i < g->n; i++) {
        bg_env* e = &g->env[i];
        if (e->terminal || e->truncated) continue;
        int64_t a = actions[i];
        if (a < 0 || a >= BG_A || !e->mask[a]) return i;
    }
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) {
        bg_env* e = &g->env[i];
        uint64_t k = orc_slot_key(slot_keys, key_state, slot0, i);
        if (e->terminal || e->truncated) { env_init(e, k); continue; }
        env_apply(e, (int)actions[i], k);
        e->truncated = (uint8_t)(!e->terminal && e->step_count >= g->max_steps);
    }
    return -1;
}

/* _observe (backgammon.py:196-206) */
void orc_bg_observe(const orc_bg* g, int64_t i, int role, float* obs) {
    const bg_env* e = &g->env[i];
    memset(obs, 0, 34 * sizeof(float));
    for (int pip = 1; pip <= 24; pip++) obs[pip - 1] = (float)signed_at(e->points, role, abs_point(role, pip));
    obs[24] = e->bar[role]; obs[25] = e->bar[1 - role];
    obs[26] = e->off[role]; obs[27] = e->off[1 - role];
    for (int j = 0; j < e->nrem; j++) obs[27 + e->rem[j]] += 1.0f;
}

void orc_bg_columns(const orc_bg* g, float* obs, uint8_t* mask, float* rewards, uint8_t* term,
                    uint8_t* trunc, int32_t* cur, int32_t* step_count, int8_t* p2r) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < g->n; i++) {
        const bg_env* e = &g->env[i];
        int fin = e->terminal || e->truncated;
        if (mask) {
            if (fin) memset(mask + i * BG_A, 0, BG_A);
            else memcpy(mask + i * BG_A, e->mask, BG_A);
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
        if (obs) orc_bg_observe(g, i, e->role_to_move, obs + (size_t)i * 34);
    }
}

/* Core.encode (backgammon.py:113-119): 24 + 7 + 4 bytes. */
int orc_bg_encode(const orc_bg* g, int64_t i, uint8_t* buf) {
    const bg_env* e = &g->env[i];
    int o = 0;
    for (int a = 0; a < 24; a++) buf[o++] = (uint8_t)((e->points[a] + 16) & 0xFF);
    buf[o++] = e->bar[0]; buf[o++] = e->bar[1]; buf[o++] = e->off[0]; buf[o++] = e->off[1];
    buf[o++] = e->role_to_move; buf[o++] = e->dice[0]; buf[o++] = e->dice[1];
    for (int j = 0; j < 4; j++) buf[o++] = j < e->nrem ? e->rem[j] : 0;
    return o;
}
