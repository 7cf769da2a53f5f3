"""Parity at the BASELINE batch sizes (2^17; shogi 2^16) through size-independent properties.

The oracle cannot replay 131,072 slots per step in seconds, but every slot's trajectory depends
only on its GLOBAL slot index (keys child(S_t, i)). So the device runs the whole batch
(the bench's fused step loop), and a sample of slots -- the first, the last and random ones -- is
replayed by the oracle with exactly those slots' keys and compared bit-exactly every step. The
fused episode counter is checked against a reduction over the WHOLE batch each step.
"""

import numpy as np
import pytest

import paper_2303_17503_b200 as bb

pytestmark = pytest.mark.gpu

COLS = ("current_player", "legal_action_mask", "rewards", "terminated", "truncated", "step_count", "player_to_role")


def _child(s, i):
    import oracle

    return oracle._child(s, i)


@pytest.mark.parametrize("game,B,steps,max_steps", [
    ("go_19x19", 1 << 17, 48, None),
    ("go_19x19", 1 << 17, 48, 20),      # truncation + auto-reset at full size
    ("chess", 1 << 17, 48, None),
    ("chess", 1 << 17, 40, 12),
    ("shogi", 1 << 16, 48, None),
    ("backgammon", 1 << 17, 96, None),
    ("go_9x9", 1 << 17, 64, None),
])
def test_full_batch_sampled_slots_match_oracle(oracle, game, B, steps, max_steps):
    import torch

    from paper_2303_17503_b200.core import resolve

    gdef = resolve(game)
    kern = gdef.batch_kernel
    limit = gdef.max_steps if max_steps is None else max_steps
    seed = 7
    root = bb.RngKey(seed)
    R = root.state
    rng = np.random.default_rng(B + steps)
    sample = np.unique(np.concatenate([[0, 1, B // 2, B - 1], rng.choice(B, 36, replace=False)])).astype(np.int64)
    idx = torch.from_numpy(sample).cuda()

    dev = torch.device("cuda", 0)
    acts = [torch.empty(B, dtype=torch.int64, device=dev) for _ in range(2)]
    eps = torch.zeros(1, dtype=torch.int64, device=dev)
    cur = kern.init(gdef, root.child(0), B, limit, device=dev, next_key=root.child(1), next_actions=acts[0])
    spare = kern.new_v(B, 0, dev, 0, limit)

    orc = oracle.make(game, len(sample), limit)
    orc.init(0, 0, [_child(_child(R, 0), int(i)) for i in sample])

    def check(v, t, with_obs):
        oc = orc.columns(with_obs=with_obs)
        for c in COLS:
            got = getattr(v.dev, c).index_select(0, idx).cpu().numpy()
            exp = oc[c]
            if got.dtype == np.bool_ or exp.dtype == np.bool_:
                got, exp = got.astype(np.uint8), exp.astype(np.uint8)
            assert np.array_equal(got, exp), f"step {t}: {c} differs at slots {sample[np.argwhere(got != exp)[:5, 0]]}"
        if with_obs:
            got = v.dev.observation.index_select(0, idx).cpu().numpy()
            assert np.array_equal(got, oc["observation"]), f"step {t}: observation differs"

    check(cur, 0, True)
    finished = 0
    for t in range(steps):
        a_key = _child(R, 2 * t + 1)
        a = acts[t % 2]
        a_s = a.index_select(0, idx).cpu().numpy()
        mask = orc.columns(with_obs=False)["legal_action_mask"]
        exp_a = np.array([oracle.random_actions(mask[k:k + 1], a_key, int(i))[0] for k, i in enumerate(sample)])
        assert np.array_equal(a_s, exp_a), f"step {t + 1}: fused random actions differ"
        nxt = kern.step(gdef, cur, a, root.child(2 * (t + 1)), limit, validate=False, out=spare,
                        next_key=root.child(2 * (t + 1) + 1), next_actions=acts[(t + 1) % 2], episodes=eps)
        spare, cur = cur, nxt
        s_key = _child(R, 2 * (t + 1))
        assert orc.step(a_s, 0, 0, [_child(s_key, int(i)) for i in sample]) == -1
        check(cur, t + 1, with_obs=(t % 8 == 7 or t == steps - 1))
        finished += int((cur.dev.terminated | cur.dev.truncated).sum())
        assert int(eps.item()) == finished, f"step {t + 1}: episode counter"
    if max_steps is not None:
        assert finished > 0
