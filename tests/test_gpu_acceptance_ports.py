"""Device ports of the reference's API-contract acceptance tests (test_acceptance.py:311-403) for
every game the device serves, chess and shogi included (the reference reserves those two ids with
no engine, so its own run covers only its nine registered games).

* mask soundness (criterion 9, test_acceptance.py:311-366): along random episodes, a masked-false
  action and an out-of-range action raise IllegalAction, a masked-true action applies. The
  reference fuzzes 1e5 states per game through the scalar API; the scalar device path costs a
  kernel launch + sync per call, so this port runs 20,000 states per game through the scalar API
  with the reference's exact key schedule, and a batched twin over 1024 slots x 64 steps that
  checks the IllegalAction slot (lowest offending live slot, tictactoe.py:111-121).
* auto-reset (criterion 10, test_acceptance.py:369-403): a slot finished in batch t is, in batch
  t+1, exactly ``init(game, skey.child(slot))`` (equal state fingerprints, step_count 0).
"""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb
from paper_2303_17503_b200.agents import random_actions

pytestmark = pytest.mark.gpu

DEVICE_GAMES = tuple(sorted(bb.available_games()))
STATES = 20000


@pytest.mark.parametrize("game_id", DEVICE_GAMES)
def test_api_contract_mask_soundness(game_id):
    spec = bb.game_spec(game_id)
    key = bb.RngKey(0xF022 + DEVICE_GAMES.index(game_id))
    checked = negative = positive = 0
    episode = 0
    while checked < STATES:
        episode += 1
        ekey = key.child(episode)
        state = bb.init(game_id, ekey.child(0))
        t = 0
        while not (state.terminated or state.truncated) and checked < STATES:
            checked += 1
            t += 1
            kk = ekey.child(2 * t)
            mask = state.legal_action_mask
            legal = np.flatnonzero(mask)
            illegal = np.flatnonzero(~mask)
            if len(illegal):
                bad = int(illegal[kk.child(1).randint(len(illegal))])
                with pytest.raises(bb.IllegalAction):
                    bb.step(state, bad, kk.child(2))
                negative += 1
            if checked % 16 == 0:
                probe = int(legal[kk.child(3).randint(len(legal))])
                bb.step(state, probe, kk.child(4))   # must not raise
                positive += 1
            if checked % 16 == 8:
                with pytest.raises(bb.IllegalAction):
                    bb.step(state, spec.num_actions, kk.child(5))
            chosen = int(legal[kk.child(0).randint(len(legal))])
            state = bb.step(state, chosen, ekey.child(2 * t + 1))
    assert checked == STATES and negative > 0 and positive > 0


@pytest.mark.parametrize("game_id", DEVICE_GAMES)
def test_batched_mask_soundness_reports_lowest_offending_slot(game_id):
    """Batched twin: per step, one random slot plays a masked-false action (or an out-of-range one
    every 4th step); batch_step must raise IllegalAction(slot = that slot) and leave the batch
    steppable; the legal actions then apply."""
    spec = bb.game_spec(game_id)
    n = 1024
    root = bb.RngKey(77)
    batch = bb.batch_init(game_id, root.child(0), n)
    rng = np.random.default_rng(5)
    for t in range(1, 65):
        acts = random_actions(batch, root.child(2 * t - 1))
        mask = batch.legal_action_mask
        live = np.flatnonzero(~(batch.terminated | batch.truncated))
        if len(live):
            slot = int(rng.choice(live))
            illegal = np.flatnonzero(~mask[slot])
            bad_acts = acts.copy()
            bad_acts[slot] = spec.num_actions if (t % 4 == 0 or not len(illegal)) else int(rng.choice(illegal))
            with pytest.raises(bb.IllegalAction) as ei:
                bb.batch_step(batch, bad_acts, root.child(2 * t))
            assert ei.value.slot == slot and ei.value.action == bad_acts[slot]
        batch = bb.batch_step(batch, acts, root.child(2 * t))


@pytest.mark.parametrize("game_id", DEVICE_GAMES)
def test_api_contract_auto_reset_per_game(game_id):
    root = bb.RngKey(8)
    n = 8 if game_id not in ("chess", "shogi", "go_19x19") else 64   # finish within the step budget
    batch = bb.batch_init(game_id, root.child(0), n)
    t = 0
    reset_checked = 0
    while reset_checked < 3 and t < 3000:
        t += 1
        actions = random_actions(batch, root.child(2 * t - 1))
        skey = root.child(2 * t)
        nxt = bb.batch_step(batch, actions, skey)
        finished = np.flatnonzero(batch.terminated | batch.truncated)
        for slot in finished:
            slot = int(slot)
            fresh = bb.init(game_id, skey.child(slot))
            assert bb.state_fingerprint(nxt.states[slot]) == bb.state_fingerprint(fresh), (game_id, t, slot)
            assert nxt.states[slot].step_count == 0
            reset_checked += 1
        batch = nxt
    assert reset_checked, f"{game_id}: no terminal observed"
