"""Device kernels vs the CPU oracle and the reference's golden trajectories.

Bit-exact bar (integer/byte work; observations are exact 0/1/count floats):
every public column, every slot's Core.encode() bytes, and the observation
tensor must be identical after every step.
"""

import numpy as np
import pytest

import goldens
import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu

COLS = ("current_player", "legal_action_mask", "rewards", "terminated", "truncated", "step_count", "player_to_role")


def compare(batch, ob, t, check_obs=True, check_encode=True):
    oc = ob.columns(with_obs=check_obs)
    for c in COLS:
        got = np.asarray(getattr(batch, c))
        exp = oc[c]
        if got.dtype == np.bool_ or exp.dtype == np.bool_:
            got, exp = got.astype(np.uint8), exp.astype(np.uint8)
        if not np.array_equal(got, exp):
            bad = np.argwhere(got != exp)[:5]
            raise AssertionError(f"step {t}: column {c} differs at {bad.tolist()}")
    if check_obs:
        got = batch.observation
        if not np.array_equal(got, oc["observation"]):
            idx = np.argwhere(got != oc["observation"])[:5]
            raise AssertionError(f"step {t}: observation differs at {idx.tolist()}")
    if check_encode:
        states = batch.states
        for i in range(batch.size):
            e = states[i].core.encode()
            if e != ob.encode(i):
                raise AssertionError(f"step {t}: slot {i} encode differs")


def _self_capture_game(game):
    from paper_2303_17503_b200.games import go

    return go.make_game(int(game.split("_")[1].split("x")[0]), allow_self_capture=True)


def _device_game(game, self_capture=False):
    from paper_2303_17503_b200.games import go

    if self_capture:
        return _self_capture_game(game)
    if game.startswith("go_") and game not in bb.available_games():   # other board sizes via make_game
        return go.make_game(int(game[3:].split("x")[0]))
    return game


def run_pair(oracle, game, n, steps, seed=0, max_steps=None, obs_every=1, enc_every=1, self_capture=False):
    sess = bb.BatchSession(_device_game(game, self_capture), n, seed, max_steps=max_steps)
    orc = oracle.Session(game, n, seed, max_steps=max_steps, self_capture=self_capture)
    compare(sess.batch, orc.b, 0)
    for t in range(1, steps + 1):
        a_dev = sess.sample_random_actions().cpu().numpy()
        a_orc = orc.sample_random_actions()
        assert np.array_equal(a_dev, a_orc), f"random actions differ at step {t}"
        sess.step(a_dev)
        assert orc.step(a_orc) == -1
        compare(sess.batch, orc.b, t, check_obs=(t % obs_every == 0), check_encode=(t % enc_every == 0))
    return sess


@pytest.mark.parametrize("game,n,steps,max_steps", [
    ("go_9x9", 32, 300, None),
    ("go_9x9", 16, 120, 20),
    ("go_19x19", 8, 560, None),
    ("go_19x19", 12, 150, 30),
    ("backgammon", 64, 600, None),
    ("backgammon", 16, 200, 25),
    ("chess", 16, 300, None),
    ("chess", 8, 120, 40),
    ("shogi", 16, 300, None),
    ("shogi", 8, 120, 40),
])
def test_device_matches_oracle(oracle, game, n, steps, max_steps):
    run_pair(oracle, game, n, steps, seed=3, max_steps=max_steps)


@pytest.mark.parametrize("game", ["go_5x5", "go_7x7", "go_11x11", "go_13x13", "go_15x15", "go_17x17"])
def test_other_go_sizes_match_oracle(oracle, game):
    """go.make_game(size) for the other instantiated sizes (go.py:114-290)."""
    run_pair(oracle, game, 24, 260, seed=5, enc_every=4)


@pytest.mark.parametrize("game,n,steps,max_steps", [("go_9x9", 64, 400, None), ("go_19x19", 16, 250, None),
                                                   ("go_9x9", 32, 150, 25)])
def test_self_capture_variant_matches_oracle(oracle, game, n, steps, max_steps):
    """make_game(allow_self_capture=True) (go.py:155-173, 249-255): suicides legal unless superko."""
    run_pair(oracle, game, n, steps, seed=11, max_steps=max_steps, self_capture=True, enc_every=5)


@pytest.mark.parametrize("name", [n for n in goldens.names() if "config1" not in n])
def test_device_matches_reference_golden(name):
    rec = goldens.load(name)
    game, n, seed, max_steps = goldens.game_args(rec)
    sess = bb.BatchSession(_device_game(game, bool(rec.get("self_capture"))), n, seed, max_steps=max_steps)
    if rec.get("init_fp"):
        assert bb.batch_fingerprint(sess.batch).hex() == rec["init_fp"]
    for t in range(rec["steps"]):
        acts = sess.sample_random_actions().cpu().numpy()
        assert goldens.digest(acts.astype(np.int64).tobytes()) == rec["act"][t], f"actions differ at step {t + 1}"
        b = sess.step(acts)
        if t < len(rec["slots"]):
            assert [bb.state_fingerprint(s).hex() for s in b.states] == rec["slots"][t], f"slots differ at {t + 1}"
        assert bb.batch_fingerprint(b).hex() == rec["fp"][t], f"batch fingerprint differs at step {t + 1}"
        if rec["obs"]:
            assert goldens.digest(b.observation.tobytes()) == rec["obs"][t], f"observations differ at step {t + 1}"


def test_baseline_config1_go9_b1024_to_all_finished():
    """BASELINE config 1: go_9x9, B=1024, seed 0, compared every step until every slot finished once."""
    rec = goldens.load("go9_config1_b1024")
    sess = bb.BatchSession("go_9x9", 1024, 0)
    done = np.zeros(1024, bool)
    for t in range(rec["steps"]):
        acts = sess.sample_random_actions().cpu().numpy()
        assert goldens.digest(acts.astype(np.int64).tobytes()) == rec["act"][t], t
        b = sess.step(acts)
        assert bb.batch_fingerprint(b).hex() == rec["fp"][t], f"step {t + 1}"
        done |= b.terminated | b.truncated
    assert done.all()


@pytest.mark.parametrize("game", ["go_9x9", "go_19x19", "backgammon", "chess", "shogi"])
def test_large_batch_vs_oracle_columns(oracle, game):
    """Thousands of slots, columns + observations checked against the oracle every step."""
    n = 2048 if game not in ("go_19x19", "chess", "shogi") else 1024
    steps = 60 if game != "backgammon" else 150
    run_pair(oracle, game, n, steps, seed=11, obs_every=10, enc_every=30)


SMALL = ["tic_tac_toe", "connect_four", "othello", "hex", "2048", "kuhn_poker", "leduc_holdem"]


@pytest.mark.parametrize("game", ["go_9x9", "go_19x19", "backgammon", "chess", "shogi"] + SMALL)
def test_batch_step_equals_scalar_steps(game):
    """Port of reference test_core.py:179-196 on the device scalar API."""
    root = bb.RngKey(71)
    n = 4
    batch = bb.batch_init(game, root.child(0), n)
    solo = [bb.init(game, root.child(0).child(i)) for i in range(n)]
    for t in range(1, 30):
        actions = bb.random_actions(batch, root.child(2 * t - 1))
        skey = root.child(2 * t)
        batch = bb.batch_step(batch, actions, skey)
        for i in range(n):
            k = skey.child(i)
            if solo[i].terminated or solo[i].truncated:
                solo[i] = bb.init(game, k)
            else:
                solo[i] = bb.step(solo[i], int(actions[i]), k)
            assert bb.state_fingerprint(solo[i]) == bb.state_fingerprint(batch.states[i]), (t, i)


def test_illegal_action_reports_lowest_slot_and_keeps_state():
    batch = bb.batch_init("go_9x9", bb.RngKey(0), 4)
    batch = bb.batch_step(batch, [40, 40, 40, 40], bb.RngKey(1))
    before = bb.batch_fingerprint(batch)
    with pytest.raises(bb.IllegalAction) as err:
        bb.batch_step(batch, [0, 1, 40, 40], bb.RngKey(2))
    assert err.value.slot == 2 and err.value.action == 40
    assert bb.batch_fingerprint(batch) == before
    with pytest.raises(bb.ShapeMismatch):
        bb.batch_step(batch, [0, 1], bb.RngKey(2))


def test_branching_previous_batch_steps_identically():
    """Immutable-batch semantics: stepping the previous batch again reproduces the same successor."""
    root = bb.RngKey(5)
    b0 = bb.batch_init("go_9x9", root.child(0), 8)
    acts = bb.random_actions(b0, root.child(1))
    b1 = bb.batch_step(b0, acts, root.child(2))
    acts2 = bb.random_actions(b1, root.child(3))
    b2 = bb.batch_step(b1, acts2, root.child(4))
    fp2 = bb.batch_fingerprint(b2)
    b2_again = bb.batch_step(b1, acts2, root.child(4))
    assert bb.batch_fingerprint(b2_again) == fp2
    assert bb.batch_fingerprint(b1) == bb.batch_fingerprint(bb.batch_step(b0, acts, root.child(2)))


@pytest.mark.parametrize("game", ["go_19x19", "backgammon", "chess", "shogi", "hex", "2048", "leduc_holdem"])
def test_slot_sharding_is_bit_identical(game):
    """Slot ranges run with slot0 offsets (one per GPU rank) equal the full batch's rows."""
    import torch
    from paper_2303_17503_b200.core import resolve

    gdef = resolve(game)
    kern = gdef.batch_kernel
    n, parts = 64, 4
    lim = gdef.max_steps
    root = bb.RngKey(9)
    full = kern.init(gdef, root.child(0), n, lim)
    shards = [kern.init(gdef, root.child(0), n // parts, lim, slot0=r * (n // parts)) for r in range(parts)]
    for t in range(1, 40):
        a = kern.random_actions(full, root.child(2 * t - 1))
        full = kern.step(gdef, full, a, root.child(2 * t), lim, validate=False)
        for r in range(parts):
            sa = kern.random_actions(shards[r], root.child(2 * t - 1))
            assert torch.equal(sa, a[r * 16:(r + 1) * 16])
            shards[r] = kern.step(gdef, shards[r], sa, root.child(2 * t), lim, validate=False)
    for r in range(parts):
        for name in ("observation", "legal_action_mask", "rewards", "current_player", "step_count"):
            assert torch.equal(getattr(shards[r].dev, name), getattr(full.dev, name)[r * 16:(r + 1) * 16]), name


@pytest.mark.parametrize("game", ["go_9x9", "go_19x19", "backgammon", "chess", "shogi"] + SMALL)
def test_fused_sampling_and_episode_counter(game):
    """Step kernels that also sample the next random actions equal the separate sampler kernel."""
    import torch
    from paper_2303_17503_b200.core import resolve

    gdef = resolve(game)
    kern = gdef.batch_kernel
    n = 96
    root = bb.RngKey(21)
    eps = torch.zeros(1, dtype=torch.int64, device="cuda")
    v = kern.init(gdef, root.child(0), n, gdef.max_steps, next_key=root.child(1))
    total = 0
    for t in range(60):
        ref = kern.random_actions(v, root.child(2 * t + 1), out=torch.empty(n, dtype=torch.int64, device="cuda"))
        assert torch.equal(v.next_actions, ref), t
        v = kern.step(gdef, v, v.next_actions, root.child(2 * (t + 1)), gdef.max_steps, validate=False,
                      next_key=root.child(2 * (t + 1) + 1), episodes=eps)
        total += int((v.dev.terminated | v.dev.truncated).sum())
    assert int(eps.item()) == total
