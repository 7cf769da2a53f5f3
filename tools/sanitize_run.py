"""Small run of every device entry point, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): per game a fused BatchSession loop (with truncation, so resets happen), validated
steps (bbk_check_actions), a branch from a predecessor batch (Go: store copy + filter rebuild),
the stand-alone sampler, observe() of the other player, device fingerprints; chess / shogi
position loads; a batched UCT search and a rollout.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py [games...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2303_17503_b200 as bb  # noqa: E402
from paper_2303_17503_b200.agents import random_actions  # noqa: E402
from paper_2303_17503_b200.core import resolve  # noqa: E402

games = sys.argv[1:] or ["go_9x9", "go_19x19", "backgammon", "chess", "shogi", "tic_tac_toe", "connect_four",
                         "othello", "hex", "2048", "kuhn_poker", "leduc_holdem"]
for g in games:
    sess = bb.BatchSession(g, 64, 1, max_steps=40, validate=False)
    for _ in range(50):
        sess.step(sess.sample_random_actions())
    root = bb.RngKey(5)
    b0 = sess.batch
    b1 = bb.batch_step(b0, random_actions(b0, root.child(1)), root.child(2))          # validated step
    b2 = bb.batch_step(b0, random_actions(b0, root.child(3)), root.child(4))          # branch from b0
    bb.batch_step(b2, random_actions(b2, root.child(5)), root.child(6))
    bb.device_fingerprints(b1)
    st = b1.states[3]
    if not (st.terminated or st.truncated):
        bb.observe(st, 0), bb.observe(st, 1)
    print(g, "ok", flush=True)

gdef = resolve("chess")
gdef.batch_kernel.load(gdef, ["r3k2r/p1ppqpb1/bn2pnp1/3PN3/1p2P3/2N2Q1p/PPPBBPPP/R3K2R w KQkq -"] * 8, key=1)
gdef = resolve("shogi")
gdef.batch_kernel.load(gdef, ["l6nl/5+P1gk/2np1S3/p1p4Pp/3P2Sp1/1PPb2P1P/P5GS1/R8/LN4bKL w RGgsn5p 1"] * 8, key=1)
print("load ok", flush=True)
b = bb.batch_init("go_9x9", bb.RngKey(2), 8)
for t in range(6):
    b = bb.batch_step(b, random_actions(b, bb.RngKey(10 + t)), bb.RngKey(20 + t))
np.asarray(bb.mcts_actions(b, bb.RngKey(3), 4))
bb.rollout("tic_tac_toe", 64, 0)
print("search/rollout ok", flush=True)
