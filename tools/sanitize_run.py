import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
"""Small fused-loop run of every game, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys

import paper_2303_17503_b200 as bb

games = sys.argv[1:] or ["go_9x9", "go_19x19", "backgammon", "chess", "shogi", "tic_tac_toe", "connect_four",
                         "othello", "hex", "2048", "kuhn_poker", "leduc_holdem"]
for g in games:
    sess = bb.BatchSession(g, 64, 1, max_steps=40, validate=False)
    for _ in range(60):
        sess.step(sess.sample_random_actions())
    bb.device_fingerprints(sess.batch)
    print(g, "ok", flush=True)
