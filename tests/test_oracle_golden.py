"""Pin the CPU oracle to the reference's own trajectories (golden fixtures).

Each fixture was produced by running the reference BatchSession
(bench.py:54-83) with random_actions (agents.py:33-46); per step it stores the
reference's batch_fingerprint (core.py:437-441) and a digest of
batch_outputs' observations (bench.py:86-97).
"""

import numpy as np
import pytest

import goldens

FAST = [n for n in goldens.names() if "config1" not in n and not n.startswith("small_")]   # small engines: no oracle, device replays them


def _replay(oracle, rec, check_obs=True, check_slots=True):
    game, n, seed, max_steps = goldens.game_args(rec)
    sess = oracle.Session(game, n, seed, max_steps=max_steps, self_capture=bool(rec.get("self_capture")))
    if rec.get("init_fp"):
        assert sess.b.batch_fingerprint().hex() == rec["init_fp"]
    for t in range(rec["steps"]):
        acts = sess.sample_random_actions()
        assert goldens.digest(acts.astype(np.int64).tobytes()) == rec["act"][t], f"actions differ at step {t + 1}"
        assert sess.step(acts) == -1
        cols = sess.b.columns(with_obs=check_obs and bool(rec["obs"]))
        if check_slots and t < len(rec["slots"]):
            fps = [f.hex() for f in sess.b.fingerprints(cols)]
            assert fps == rec["slots"][t], f"slot fingerprints differ at step {t + 1}"
        assert sess.b.batch_fingerprint(cols).hex() == rec["fp"][t], f"batch fingerprint differs at step {t + 1}"
        if check_obs and rec["obs"]:
            assert goldens.digest(cols["observation"].tobytes()) == rec["obs"][t], f"observations differ at step {t + 1}"


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference_golden(oracle, name):
    _replay(oracle, goldens.load(name))


@pytest.mark.slow
def test_oracle_matches_baseline_config1(oracle):
    """BASELINE config 1: go_9x9, 1024 envs, seed 0, until every slot finished once (379 steps)."""
    rec = goldens.load("go9_config1_b1024")
    _replay(oracle, rec, check_obs=False, check_slots=False)
