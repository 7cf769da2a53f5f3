/* bbk.h -- C-ABI of the B200 batched board-game step (libbbk.so).
 *
 * This is the drop-in boundary for the reference's batch-kernel plugin
 * protocol, `GameDef.batch_kernel` (reference pkg/src/boardbatch/core.py:88),
 * whose three calls are
 *     kern.init(gdef, key, n, limit)            core.py:346-348
 *     kern.step(gdef, v, acts, key, limit)      core.py:366-368
 *     kern.state_at(gdef, v, i, limit)          core.py:276-282
 * (reference implementation: games/tictactoe.py:71-198). Every entry point
 * below takes plain device pointers and sizes (no torch types), runs
 * asynchronously on `stream` (a cudaStream_t, NULL = legacy default), and
 * returns 0 or a cudaError_t. The host mirror of the protocol lives in
 * paper_2303_17503_b200/games/*.py and binds these symbols with ctypes.
 *
 * Key contract (core.py:374, tictactoe.py:99-106): slot i uses
 * k_i = child(key_state, slot0 + i) with child(k, j) = mix64(k + (j+1)*phi)
 * (rng.py:43-45), or k_i = slot_keys[i] when slot_keys != NULL (the scalar
 * init/step path, core.py:223-243). A reset draws the player permutation
 * from child(k_i, 0) % 2 and the core from child(k_i, 1) (core.py:227-228).
 *
 * Layouts (row-major, batch leading, SURVEY §8a dtypes):
 *   observation        float32 [n, *obs_shape]  current player's view
 *   legal_action_mask  uint8   [n, A]           zero when finished
 *   rewards            float32 [n, P]           indexed by player (P = 2; the one-player 2048: 1)
 *   terminated, truncated uint8 [n]
 *   current_player, step_count int32 [n]
 *   player_to_role     int8    [n, P]
 */
#ifndef BBK_H
#define BBK_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBK_ABI_VERSION 6   /* 3: fingerprints, small engines; 4: batched UCT search;
                               5: per-size Go superko filters (bbk_go_filter_words, size arg of bbk_go_rebuild_bloom);
                               6: Go chain labels moved from bbk_go_state to the in-place bbk_go_store, bbk_go_relabel */

typedef struct bbk_cols {
    float*    observation;        /* may be NULL: skip observation emission */
    uint8_t*  legal_action_mask;
    float*    rewards;
    uint8_t*  terminated;
    uint8_t*  truncated;
    int32_t*  current_player;
    int32_t*  step_count;
    int8_t*   player_to_role;
    /* Optional fused outputs of an init/step call (ignored in `in` columns):
     *   next_actions[n]  agents.random_actions(new batch, next_key) (agents.py:33-46),
     *                    sampled from the new legal mask while it is still on chip,
     *                    so the benchmark loop needs no separate sampling pass;
     *   episodes         += number of finished slots (bench.py:129). */
    int64_t*  next_actions;
    uint64_t  next_key;
    unsigned long long* episodes;
} bbk_cols;

/* ------------------------------------------------------------------ Go --
 * Replaces games/go.py (make_game(size), go.py:114-290): apply :219-262,
 * legal_mask :121-174 (positional superko), score_rewards :176-210,
 * observe :264-273, Core.encode :103-111.
 *   pat[n, pat_stride]  uint16: bit 2t / 2t+1 = black / white stone at the
 *                       point in boards_hist[t] (t = 0 newest .. 7)
 *   store.lab[n, pat_stride] uint16: chain label per stone = one point of the stone's chain,
 *                       maintained IN PLACE along a lineage like the history (a step writes only
 *                       the labels it changes; values at empty points are never read), rebuilt
 *                       from a batch's board by bbk_go_relabel when that batch branches
 *   history[n, hist_cap] uint64 append-only superko hashes (history set)
 *   bloom[n, bbk_go_filter_words(size)] uint32: a Bloom filter over history hashes, then a
 *                        filter of the (black, white) stone-count pairs of the history
 *                        positions (a repeat must have equal counts). Sized per board:
 *                        2048 + 2048 bits up to 9x9, 4096 + 2048 up to 13x13, else the
 *                        8192 + 2048 bits below (the largest).
 */
#define BBK_GO_BLOOM_WORDS 256
#define BBK_GO_PAIR_WORDS 64
#define BBK_GO_FILTER_WORDS (BBK_GO_BLOOM_WORDS + BBK_GO_PAIR_WORDS)

typedef struct bbk_go_state {
    uint16_t* pat;
    uint64_t* hash;
    uint64_t* hist_xor;
    int32_t*  hist_len;
    uint8_t*  role_to_move;
    uint8_t*  pass_count;
} bbk_go_state;

typedef struct bbk_go_store {
    uint64_t* history;
    uint32_t* bloom;
    uint16_t* lab;      /* [n, pat_stride] chain label of every stone (a point of its chain), in place */
    int32_t   hist_cap;
} bbk_go_store;

int bbk_go_pat_stride(int size);
/* uint32 words of one env's superko filter row (-1 for an unsupported size) */
int bbk_go_filter_words(int size);

/* batch_init (core.py:340-350) */
int bbk_go_init(int size, const bbk_cols* out, const bbk_go_state* out_s, const bbk_go_store* store,
                int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                int32_t max_steps, void* stream);

/* batch_step (core.py:353-386): auto-reset of finished slots, else go.apply.
 * allow_self_capture: make_game(allow_self_capture=True) (go.py:155-173, 249-255).
 * Actions are assumed legal (validate first with bbk_check_actions). */
int bbk_go_step(int size, double komi, int allow_self_capture, const bbk_cols* in, const bbk_go_state* in_s,
                const bbk_cols* out, const bbk_go_state* out_s, const bbk_go_store* store,
                const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state,
                const uint64_t* slot_keys, int32_t max_steps, void* stream);

/* observe(state, player) (core.py:246-251) for an explicit role per slot. */
int bbk_go_observe(int size, const uint16_t* pat, const uint8_t* role, float* obs, int64_t n, void* stream);

/* Rebuild Bloom filters from history[0:hist_len) (used when a batch branches). */
int bbk_go_rebuild_bloom(int size, const bbk_go_store* store, const int32_t* hist_len, int64_t n, void* stream);
/* Rebuild the chain labels of store.lab from each board's current position (bits 0/1 of pat):
 * label = the lowest point of the chain. Used with bbk_go_rebuild_bloom when a batch branches. */
int bbk_go_relabel(int size, const bbk_go_store* store, const uint16_t* pat, int64_t n, void* stream);

/* ---------------------------------------------------------- Backgammon --
 * Replaces games/backgammon.py: _legal_mask :62-95, _roll :125-130,
 * _final :137-147, _apply :150-193, _observe :196-206, encode :113-119. */
typedef struct bbk_bg_state {
    int8_t*   points;     /* [n, 24] signed, + = role 0 */
    uint8_t*  misc;       /* [n, 12]: bar0 bar1 off0 off1 role d1 d2 rem0..3 nrem */
} bbk_bg_state;

int bbk_bg_init(const bbk_cols* out, const bbk_bg_state* out_s, int64_t n, int64_t slot0,
                uint64_t key_state, const uint64_t* slot_keys, int32_t max_steps, void* stream);
int bbk_bg_step(const bbk_cols* in, const bbk_bg_state* in_s, const bbk_cols* out, const bbk_bg_state* out_s,
                const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state,
                const uint64_t* slot_keys, int32_t max_steps, void* stream);
int bbk_bg_observe(const bbk_bg_state* s, const uint8_t* role, float* obs, int64_t n, void* stream);

/* --------------------------------------------------------------- Chess --
 * No reference engine (reserved spec, games/__init__.py:23); rules and
 * encodings per PAPER.md:781-856 and DESIGN.md §3.3 (CPU twin:
 * oracle/orc_chess.c, perft-pinned).
 *   board[n, 64]  piece code per square (a1 = 0; colour << 3 | P1 N2 B3 R4 Q5 K6)
 *   misc[n, 8]    stm, castling bits, ep square (255 = none), half-move clock, repetition
 *   hist[n, 4608] per-env ring of 128 plies: packed boards (32 B) + meta (u32),
 *                 shared along a trajectory (in place). */
typedef struct bbk_chess_state {
    uint8_t* board;
    uint8_t* misc;
    uint8_t* hist;
} bbk_chess_state;

int bbk_chess_init(const bbk_cols* out, const bbk_chess_state* out_s, int64_t n, int64_t slot0, uint64_t key_state,
                   const uint64_t* slot_keys, int32_t max_steps, void* stream);
/* Start slots from given positions (a reset with the position instead of the initial one; history
 * empty, step_count 0, player_to_role from the slot key as in init). boards [n,64] piece codes,
 * misc [n,8] = stm, castling bits, en-passant square (int8, -1 none), half-move clock. No reference
 * interface (chess has no reference engine): the device twin of oracle/orc_chess.c orc_chess_set_fen,
 * used by the device perft / rule-position tests. */
int bbk_chess_load(const bbk_cols* out, const bbk_chess_state* out_s, const uint8_t* boards, const uint8_t* misc,
                   int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys, int32_t max_steps,
                   void* stream);
int bbk_chess_step(const bbk_cols* in, const bbk_chess_state* in_s, const bbk_cols* out, const bbk_chess_state* out_s,
                   const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                   int32_t max_steps, void* stream);
int bbk_chess_observe(const bbk_chess_state* s, const int32_t* step_count, const uint8_t* role, float* obs, int64_t n,
                      void* stream);

/* --------------------------------------------------------------- Shogi --
 * No reference engine (reserved spec, games/__init__.py:31); rules and
 * encodings per PAPER.md:1278-1354 and DESIGN.md §3.4 (CPU twin:
 * oracle/orc_shogi.c, perft-pinned).
 *   board[n, 96]  absolute piece codes (owner << 4 | FU1 KY2 KE3 GI4 KI5 KA6 HI7 OU8 TO..RY 9-14), 81 used
 *   misc[n, 16]   hands[2][7] (FU KY KE GI KI KA HI), side to move, repetition count
 *   hist[n, hist_cap] u64 position keys by ply (four-fold repetition), shared in place. */
typedef struct bbk_shogi_state {
    uint8_t*  board;
    uint8_t*  misc;
    uint64_t* hist;
    int32_t   hist_cap;
} bbk_shogi_state;

int bbk_shogi_init(const bbk_cols* out, const bbk_shogi_state* out_s, int64_t n, int64_t slot0, uint64_t key_state,
                   const uint64_t* slot_keys, int32_t max_steps, void* stream);
/* As bbk_chess_load: boards [n,96] absolute codes (owner << 4 | type, squares r*9+c), misc [n,16] =
 * hands [2][7] (FU KY KE GI KI KA HI), side to move. Twin of oracle orc_shogi_set_sfen. */
int bbk_shogi_load(const bbk_cols* out, const bbk_shogi_state* out_s, const uint8_t* boards, const uint8_t* misc,
                   int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys, int32_t max_steps,
                   void* stream);
int bbk_shogi_step(const bbk_cols* in, const bbk_shogi_state* in_s, const bbk_cols* out, const bbk_shogi_state* out_s,
                   const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                   int32_t max_steps, void* stream);
int bbk_shogi_observe(const bbk_shogi_state* s, const int32_t* step_count, const uint8_t* role, float* obs, int64_t n,
                      void* stream);

/* ------------------------------------------------------------- generic --
 * agents.random_actions (agents.py:33-46): a_i = index of the d-th legal
 * action, d = child(key, slot0+i) % max(popcount(mask_i), 1); 0 if none. */
int bbk_random_actions(const uint8_t* mask, int64_t n, int32_t num_actions, uint64_t key_state,
                       int64_t slot0, int64_t* actions, void* stream);

/* IllegalAction check (core.py:234-239, tictactoe.py:111-121): writes the
 * lowest live slot whose action is out of range or masked out into
 * *first_bad, or INT32_MAX when every live action is legal (a plain store:
 * no initialisation needed); finished slots are exempt. One launch. */
int bbk_check_actions(const uint8_t* mask, const uint8_t* terminated, const uint8_t* truncated,
                      const int64_t* actions, int64_t n, int32_t num_actions, int32_t* first_bad,
                      void* stream);

/* Sum of (terminated | truncated) over n slots, added into *count
 * (bench.py:129 episode counter). */
int bbk_count_finished(const uint8_t* terminated, const uint8_t* truncated, int64_t n,
                       unsigned long long* count, void* stream);

/* The host read of a step's results (bench.py:121-129 reads rewards / flags every step): after the
 * work queued on `main_stream`, `count` (<= 8) device -> host copies dst[i] <- src[i] (bytes[i])
 * on `copy_stream`, then `done` recorded on it. `after` and `done` are cudaEvent_t handles the
 * caller owns. One call instead of an event record, a stream wait, per-buffer copies and a record. */
int bbk_fetch_async(int count, void* const* dst, const void* const* src, const int64_t* bytes,
                    void* main_stream, void* copy_stream, void* after, void* done);

int bbk_abi_version(void);
const char* bbk_build_info(void);

/* Checked builds (-DBBK_CHECKS=1, tools/checked_build.sh): 1 if this library records failed
 * scratch-index / capacity checks. bbk_debug_failures writes, per translation unit (go, chess,
 * shogi, backgammon, small, mcts, fingerprint, util), (first failing source line << 32) | count,
 * optionally clears them, and returns how many units recorded a failure (always 0 unchecked). */
int bbk_debug_checks(void);
int bbk_debug_failures(int reset, unsigned long long* out, int n);

/* Batched rollouts (agents.py:113-116 over a batch): after each step, record every slot's first
 * finished episode -- returns [n, players] by player and its length -- into done / returns /
 * lengths, and add the number of newly finished slots to *count. */
int bbk_latch_finished(const uint8_t* terminated, const uint8_t* truncated, const float* rewards,
                       const int32_t* step_count, int players, int64_t n, uint8_t* done, float* returns,
                       int32_t* lengths, unsigned long long* count, void* stream);

/* ------------------------------------------------------- small engines --
 * The reference's other engines, one thread per slot:
 * game 0 tic_tac_toe (games/tictactoe.py), 1 connect_four (connect_four.py),
 * 2 othello (othello.py), 3 hex (hexgame.py), 4 2048 (play2048.py),
 * 5 kuhn_poker (kuhn_poker.py), 6 leduc_holdem (leduc_holdem.py).
 * Per-slot Core in a BBK_SMALL_STATE_BYTES blob [n, 48] (layouts in
 * csrc/small.cuh). Columns as above, except that the one-player 2048 has
 * rewards [n, 1] and player_to_role [n, 1]. */
#define BBK_SMALL_STATE_BYTES 48
int bbk_small_state_bytes(void);
int bbk_small_init(int game, const bbk_cols* out, uint8_t* out_blob, int64_t n, int64_t slot0, uint64_t key_state,
                   const uint64_t* slot_keys, int32_t max_steps, void* stream);
int bbk_small_step(int game, const bbk_cols* in, const uint8_t* in_blob, const bbk_cols* out, uint8_t* out_blob,
                   const int64_t* actions, int64_t n, int64_t slot0, uint64_t key_state, const uint64_t* slot_keys,
                   int32_t max_steps, void* stream);
int bbk_small_observe(int game, const uint8_t* blob, const uint8_t* terminated, const uint8_t* role, float* obs,
                      int64_t n, void* stream);

/* ------------------------------------------------- state fingerprints --
 * Device-side core.state_fingerprint (core.py:417-434) for every slot of a
 * batch: out[n, 16] = blake2b-16 of
 *   game_id | <iiBB>(current_player, step_count, terminated, truncated)
 *   | player_to_role | rewards f32[P] | packbits(mask, MSB first) | Core.encode().
 * `scratch` is [n, stride] bytes (stride = bbk_fingerprint_stride), `lens` [n].
 * batch_fingerprint (core.py:437-441) is blake2b over out[0..n) in slot order.
 * game_code: 0 Go (size = board size), 1 backgammon, 2 chess, 3 shogi, 4 small engines. */
int bbk_fingerprint_stride(int game_code, int size);
int bbk_go_fingerprint(int size, const bbk_cols* cols, const bbk_go_state* s, int64_t n, uint8_t* scratch,
                       int64_t stride, int32_t* lens, uint8_t* out, void* stream);
int bbk_bg_fingerprint(const bbk_cols* cols, const bbk_bg_state* s, int64_t n, uint8_t* scratch, int64_t stride,
                       int32_t* lens, uint8_t* out, void* stream);
int bbk_chess_fingerprint(const bbk_cols* cols, const bbk_chess_state* s, int64_t n, uint8_t* scratch,
                          int64_t stride, int32_t* lens, uint8_t* out, void* stream);
int bbk_shogi_fingerprint(const bbk_cols* cols, const bbk_shogi_state* s, int64_t n, uint8_t* scratch,
                          int64_t stride, int32_t* lens, uint8_t* out, void* stream);
int bbk_small_fingerprint(int game, const bbk_cols* cols, const uint8_t* blob, int64_t n, uint8_t* scratch,
                          int64_t stride, int32_t* lens, uint8_t* out, void* stream);
/* Host build of the same blake2b-16 (pinned against hashlib by the CPU tests). */
int bbk_blake2b16_host(const uint8_t* msg, int64_t len, uint8_t* out);

/* ------------------------------------------------ batched UCT search --
 * agents.mcts_agent (reference agents.py:49-131) for a batch of root states,
 * one search per root, all searches advancing one simulation at a time
 * (SURVEY §8f rank 3). The host owns the loop: per simulation
 *   bbk_mcts_select -> bbk_copy_rows (pool -> staging) -> the game's step
 *   kernel -> bbk_copy_rows (staging -> pool) -> bbk_mcts_untried ->
 *   rollout: { bbk_mcts_rollout_actions -> step -> bbk_mcts_latch }* ->
 *   bbk_mcts_backup,
 * then bbk_mcts_best. The node pool is an ordinary batch of n_search *
 * max_nodes slots of the game's state; node k of search s is pool row
 * s * max_nodes + k. Each search draws from its own MT19937 stream seeded
 * like Python's random.Random(key_state) (agents.py:85), in the reference's
 * order, so the chosen actions are the reference's. All arrays are device
 * memory, [n_search][max_nodes] unless noted. */
typedef struct bbk_mcts_tree {
    int64_t   n_search;
    int32_t   max_nodes;       /* simulations + 1 */
    int32_t   num_actions;     /* A */
    int32_t   mask_words;      /* ceil(A / 32) */
    uint32_t* mt;              /* [n_search][625]: Twister words, then the index */
    int32_t*  visits;
    double*   value_sum;
    int32_t*  parent;
    int32_t*  first_child;
    int32_t*  last_child;
    int32_t*  next_sibling;
    int32_t*  action;          /* action leading to the node (-1 at the root) */
    uint8_t*  role;            /* role to move at the node */
    uint32_t* untried;         /* [n_search][max_nodes][mask_words] untried-action bitset */
    int32_t*  untried_count;
    int32_t*  next_node;       /* [n_search] */
    int32_t*  leaf;            /* [n_search] node the current simulation ends at */
} bbk_mcts_tree;

/* Seed every search's Twister from key_states[n_search] (u64) and create its root. */
int bbk_mcts_seed(const bbk_mcts_tree* t, const uint64_t* key_states, void* stream);
/* Untried set and role of node[s] (node == NULL: the root) of every search from
 * staging row s's mask / current_player / player_to_role; node[s] < 0 skips. */
int bbk_mcts_untried(const bbk_mcts_tree* t, const uint8_t* mask, const int32_t* current_player,
                     const int8_t* player_to_role, const int32_t* node, void* stream);
/* Selection + expansion (agents.py:89-109) with exploration constant c and
 * log_table[v] = log(v) for v <= max_nodes. Outputs per search: src_row (pool
 * row to step from), dst_row (pool row of the new child, -1 if the selected node
 * is finished), actions, new_node (-1 likewise). */
int bbk_mcts_select(const bbk_mcts_tree* t, double c, const double* log_table, int32_t* src_row, int32_t* dst_row,
                    int64_t* actions, int32_t* new_node, void* stream);
/* Rollout moves (agents.py:113-116) from staging masks [n_search, A]; done[s] != 0: lowest legal. */
int bbk_mcts_rollout_actions(const bbk_mcts_tree* t, const uint8_t* mask, const uint8_t* done, int64_t* actions,
                             void* stream);
/* Role rewards of rollouts that just ended (agents.py:117, 126-131) into role_returns [n, 2];
 * sel != NULL restricts to slots with (sel[s] >= 0) == (want != 0). */
int bbk_mcts_latch(const uint8_t* terminated, const uint8_t* truncated, const float* rewards,
                   const int8_t* player_to_role, const int32_t* sel, int want, int64_t n, uint8_t* done,
                   float* role_returns, unsigned long long* count, void* stream);
/* Backup (agents.py:117-122): value_sum += scale * role_return[mover] + offset along each path. */
int bbk_mcts_backup(const bbk_mcts_tree* t, const float* role_returns, double scale, double offset, void* stream);
/* Most visited root child, ties to the lowest action (agents.py:124-129). */
int bbk_mcts_best(const bbk_mcts_tree* t, int64_t* actions, void* stream);

/* Row gather / scatter of up to BBK_ROW_COPY_MAX per-slot tensors at once:
 * dst[dst_idx[i]] = src[src_idx[i]] (index NULL = i; a negative index skips
 * row i), rows of row_bytes moved in units of `unit` (1, 4, 8 or 16) bytes. */
#define BBK_ROW_COPY_MAX 24
typedef struct bbk_row_copy {
    const void* src;
    void*       dst;
    int64_t     row_bytes;
    int64_t     unit;
} bbk_row_copy;
typedef struct bbk_row_copy_set {
    int32_t      count;
    bbk_row_copy t[BBK_ROW_COPY_MAX];
} bbk_row_copy_set;
int bbk_copy_rows(const bbk_row_copy_set* set, const int32_t* src_idx, const int32_t* dst_idx, int64_t n,
                  void* stream);
/* Host twin of the device Twister (CPU tests against Python's random):
 * out[i] = randrange(below[i]) on random.Random(seed), or a raw 32-bit word when below[i] == 0. */
int bbk_mt19937_host(uint64_t seed, const uint32_t* below, int64_t n, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
