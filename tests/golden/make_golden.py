"""Generate golden trajectory fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``boardbatch`` from /root/reference/pkg/src (read-only) and drives
``BatchSession`` (reference bench.py:54-83) with ``random_actions``
(agents.py:33-46). Per step it records the reference's own
``batch_fingerprint`` (core.py:437-441), a blake2b of the
``batch_outputs`` observations (bench.py:86-97) and of the actions. The
fixtures travel with the repo; the GPU box never needs the reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(b: bytes) -> str:
    return hashlib.blake2b(b, digest_size=16).hexdigest()


def record(name, game, n, seed, steps, max_steps=None, per_slot_steps=0, obs=True):
    import numpy as np
    import boardbatch as bb
    from boardbatch.bench import BatchSession, batch_outputs

    t0 = time.time()
    sess = BatchSession(game, n, seed, max_steps=max_steps)
    gdef = sess.gdef
    rec = {
        "name": name,
        "game_id": gdef.game_id,
        "size": gdef.spec.observation_shape[0] if gdef.game_id.startswith("go_") else None,
        "batch": n,
        "seed": seed,
        "steps": steps,
        "max_steps": sess.batch.max_steps,
        "generator": "tests/golden/make_golden.py (reference boardbatch %s)" % bb.__version__,
        "init_fp": sess.batch and bb.batch_fingerprint(sess.batch).hex(),
        "init_obs": _digest(batch_outputs(sess.batch)["observations"].tobytes()) if obs else None,
        "fp": [],
        "obs": [],
        "act": [],
        "episodes": [],
        "slots": [],
    }
    eps = 0
    for t in range(steps):
        acts = sess.sample_random_actions()
        batch = sess.step(acts)
        rec["fp"].append(bb.batch_fingerprint(batch).hex())
        rec["act"].append(_digest(np.asarray(acts, dtype=np.int64).tobytes()))
        if obs:
            rec["obs"].append(_digest(batch_outputs(batch)["observations"].tobytes()))
        eps += int((batch.terminated | batch.truncated).sum())
        rec["episodes"].append(eps)
        if t < per_slot_steps:
            rec["slots"].append([bb.state_fingerprint(s).hex() for s in batch.states])
    rec["seconds"] = round(time.time() - t0, 1)
    return rec


def record_until_all_finished(name, game, n, seed):
    """BASELINE config 1: run until every slot has finished once."""
    import numpy as np
    import boardbatch as bb
    from boardbatch.bench import BatchSession

    t0 = time.time()
    sess = BatchSession(game, n, seed)
    done = np.zeros(n, bool)
    fps, acts_d = [], []
    while not done.all():
        acts = sess.sample_random_actions()
        batch = sess.step(acts)
        done |= batch.terminated | batch.truncated
        fps.append(bb.batch_fingerprint(batch).hex())
        acts_d.append(_digest(np.asarray(acts, dtype=np.int64).tobytes()))
    return {
        "name": name, "game_id": game, "size": 9, "batch": n, "seed": seed, "steps": len(fps),
        "max_steps": sess.batch.max_steps,
        "generator": "tests/golden/make_golden.py (reference boardbatch %s)" % bb.__version__,
        "init_fp": None, "init_obs": None, "fp": fps, "obs": [], "act": acts_d, "episodes": [], "slots": [],
        "seconds": round(time.time() - t0, 1),
    }


def main():
    sys.path.insert(0, REF)
    import boardbatch as bb  # noqa: F401
    from boardbatch.games import go

    go19 = go.make_game(19)
    jobs = [
        ("go9_s0_b16", lambda: record("go9_s0_b16", "go_9x9", 16, 0, 400, per_slot_steps=40)),
        ("go9_s99_b8_trunc20", lambda: record("go9_s99_b8_trunc20", "go_9x9", 8, 99, 120, max_steps=20, per_slot_steps=25)),
        ("go19_s0_b4", lambda: record("go19_s0_b4", go19, 4, 0, 1100, per_slot_steps=10)),
        ("go19_s2718_b6_trunc40", lambda: record("go19_s2718_b6_trunc40", go19, 6, 2718, 130, max_steps=40)),
        ("bg_s0_b16", lambda: record("bg_s0_b16", "backgammon", 16, 0, 1500, per_slot_steps=40)),
        ("bg_s99_b8_trunc50", lambda: record("bg_s99_b8_trunc50", "backgammon", 8, 99, 300, max_steps=50)),
        ("go9_config1_b1024", lambda: record_until_all_finished("go9_config1_b1024", "go_9x9", 1024, 0)),
        ("go7_s0_b16", lambda: record("go7_s0_b16", go.make_game(7), 16, 0, 200, per_slot_steps=10)),
        ("go13_s1_b8", lambda: record("go13_s1_b8", go.make_game(13), 8, 1, 250, per_slot_steps=10)),
        # make_game(allow_self_capture=True) (go.py:155-173, 249-255): suicide moves legal unless superko
        ("go9sc_s0_b16", lambda: dict(record("go9sc_s0_b16", go.make_game(9, allow_self_capture=True), 16, 0, 300,
                                             per_slot_steps=30), self_capture=True)),
        ("go19sc_s5_b4_trunc120", lambda: dict(record("go19sc_s5_b4_trunc120", go.make_game(19, allow_self_capture=True),
                                                      4, 5, 150, max_steps=120), self_capture=True)),
    ]
    only = set(sys.argv[1:])
    for name, fn in jobs:
        if only and name not in only:
            continue
        rec = fn()
        path = os.path.join(HERE, name + ".json")
        with open(path, "w") as fh:
            json.dump(rec, fh, separators=(",", ":"))
        print(f"{name}: {rec['steps']} steps in {rec['seconds']} s -> {os.path.getsize(path)} bytes", flush=True)


if __name__ == "__main__":
    main()
