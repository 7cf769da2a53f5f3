"""Golden UCT-search decisions made by running the REFERENCE's own ``agents.mcts_agent``
(agents.py:63-123) in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mcts.py [names...]

Each job builds roots with the reference ``BatchSession`` (random play for ``t`` steps), then
records, for every slot i, ``mcts_agent(states[i], RngKey(key_seed).child(i), sims, ...)`` (0 for
a finished slot) -- the key convention of the device's batched ``mcts_actions``. The batch
fingerprint of the roots is stored too, so the replay can check it searched the same states.
Replayed by tests/test_gpu_search.py.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# name, game, n, seed, t, sims, key_seed, exploration, value_transform, max_steps
JOBS = [
    ("mcts_tic_tac_toe_s0_b32_t2", "tic_tac_toe", 32, 0, 2, 16, 7, None, None, None),
    ("mcts_tic_tac_toe_s1_b16_t0", "tic_tac_toe", 16, 1, 0, 64, 11, None, None, None),
    ("mcts_connect_four_s0_b16_t4", "connect_four", 16, 0, 4, 32, 5, None, None, None),
    ("mcts_connect_four_s3_b8_t6_vt", "connect_four", 8, 3, 6, 24, 9, 1.0, (2.0, 0.3), None),
    ("mcts_othello_s0_b8_t10", "othello", 8, 0, 10, 8, 3, None, None, None),
    ("mcts_hex_s0_b8_t5", "hex", 8, 0, 5, 8, 4, None, None, None),
    ("mcts_go_5x5_s0_b8_t6", "go_5x5", 8, 0, 6, 12, 2, None, None, None),
    ("mcts_go_9x9_s0_b4_t20", "go_9x9", 4, 0, 20, 4, 1, None, None, None),
    ("mcts_go_9x9_s99_b4_t10_trunc40", "go_9x9", 4, 99, 10, 6, 8, None, None, 40),
    ("mcts_go_9x9_s0_b8_t20_sims16", "go_9x9", 8, 0, 20, 16, 1, None, None, None),
    ("mcts_go_19x19_s0_b2_t20", "go_19x19", 2, 0, 20, 4, 1, None, None, None),
    ("mcts_hex_s2_b16_t9_sims32", "hex", 16, 2, 9, 32, 6, None, None, None),
    ("mcts_othello_s5_b16_t30_sims24", "othello", 16, 5, 30, 24, 12, None, None, None),
    ("mcts_tic_tac_toe_s2_b64_t4_sims256", "tic_tac_toe", 64, 2, 4, 256, 13, None, None, None),
]


# match jobs: name, game, agents ("random" | sims), games_per_pair, key_seed
MATCHES = [
    ("mcts_matches_tic_tac_toe_k4", "tic_tac_toe", ["random", 8, 16], 6, 4),
    ("mcts_matches_connect_four_k9", "connect_four", [16, "random"], 10, 9),
    ("mcts_matches_hex_k2", "hex", [4, "random"], 4, 2),
    ("mcts_matches_othello_k1", "othello", ["random", "random"], 20, 1),
    ("mcts_matches_backgammon_k3", "backgammon", ["random", "random"], 6, 3),
    ("mcts_matches_kuhn_poker_k5", "kuhn_poker", ["random", "random"], 40, 5),
    ("mcts_matches_go_9x9_k7", "go_9x9", [2, "random"], 3, 7),
]


def record_matches(name, game, agents, games, key_seed):
    import boardbatch as bb
    from boardbatch.agents import mcts_policy, play_game, random_policy, run_matches
    from boardbatch.core import resolve as ref_resolve

    t0 = time.time()
    pol = [random_policy() if a == "random" else mcts_policy(a) for a in agents]
    gdef = ref_resolve(resolve(game))
    res = run_matches(gdef, pol, games, bb.RngKey(key_seed))
    # every game's final (rewards, step_count), pairings in run_matches order (agents.py:195-214)
    per_game = []
    k = 0
    for i in range(len(pol)):
        for j in range(i + 1, len(pol)):
            pair_key = bb.RngKey(key_seed).child(k)
            k += 1
            finals = [play_game(gdef, (pol[i], pol[j]), pair_key.child(g)) for g in range(games)]
            per_game.append([[float(f.rewards[0]), float(f.rewards[1]), int(f.step_count)] for f in finals])
    return {
        "name": name, "game": game, "agents": agents, "games_per_pair": games, "key_seed": key_seed,
        "results": [[r.game_id, r.agent_a, r.agent_b, r.wins_a, r.wins_b, r.draws] for r in res],
        "games": per_game,
        "generator": "tests/golden/make_golden_mcts.py (reference boardbatch %s)" % bb.__version__,
        "seconds": round(time.time() - t0, 1),
    }


def resolve(game):
    from boardbatch.games import go

    if game.startswith("go_") and game != "go_9x9":
        return go.make_game(int(game[3:].split("x")[0]))
    return game


def record(name, game, n, seed, t, sims, key_seed, exploration, vt, max_steps):
    import boardbatch as bb
    from boardbatch.agents import mcts_agent
    from boardbatch.bench import BatchSession

    t0 = time.time()
    sess = BatchSession(resolve(game), n, seed, max_steps=max_steps)
    for _ in range(t):
        sess.step(sess.sample_random_actions())
    batch = sess.batch
    key = bb.RngKey(key_seed)
    kw = {}
    if exploration is not None:
        kw["exploration"] = exploration
    if vt is not None:
        kw["value_transform"] = tuple(vt)
    actions = []
    for i, st in enumerate(batch.states):
        if st.terminated or st.truncated:
            actions.append(0)
        else:
            actions.append(int(mcts_agent(st, key.child(i), sims, **kw)))
    return {
        "name": name, "game": game, "batch": n, "seed": seed, "t": t, "sims": sims, "key_seed": key_seed,
        "exploration": math.sqrt(2.0) if exploration is None else exploration,
        "value_transform": list(vt) if vt is not None else [1.0, 0.0],
        "max_steps": max_steps, "roots_fp": bb.batch_fingerprint(batch).hex(), "actions": actions,
        "generator": "tests/golden/make_golden_mcts.py (reference boardbatch %s)" % bb.__version__,
        "seconds": round(time.time() - t0, 1),
    }


def main():
    sys.path.insert(0, REF)
    only = set(sys.argv[1:])
    for job in JOBS:
        if only and job[0] not in only:
            continue
        rec = record(*job)
        path = os.path.join(HERE, job[0] + ".json")
        with open(path, "w") as fh:
            json.dump(rec, fh, separators=(",", ":"))
        print(f"{job[0]}: {rec['actions']} in {rec['seconds']} s", flush=True)
    for job in MATCHES:
        if only and job[0] not in only:
            continue
        rec = record_matches(*job)
        path = os.path.join(HERE, job[0] + ".json")
        with open(path, "w") as fh:
            json.dump(rec, fh, separators=(",", ":"))
        print(f"{job[0]}: {rec['results']} in {rec['seconds']} s", flush=True)


if __name__ == "__main__":
    main()
