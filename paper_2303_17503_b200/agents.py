"""Agents (reference agents.py): random sampling, batched rollouts, UCT search and matches on the device."""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .core import EnvState, TerminalStep
from .rng import RngKey


def random_agent(state: EnvState, key: RngKey) -> int:
    """Uniform draw over the mask-true actions (agents.py:25-30)."""
    if state.terminated or state.truncated:
        raise TerminalStep("cannot pick an action in a finished state")
    legal = np.flatnonzero(state.legal_action_mask)
    return int(legal[key.randint(len(legal))])


def random_actions_device(batch, key: RngKey, out=None):
    """Per-slot uniform legal actions as a CUDA int64 tensor (no host copy).

    Slot i receives exactly ``random_agent(states[i], key.child(slot0 + i))``;
    finished slots get 0 (agents.py:33-46), computed by bbk_random_actions.
    """
    v = batch._v
    if out is None and v.next_actions is not None and v.next_key == key.state:
        return v.next_actions   # already sampled by the fused step/init kernel from the same mask and key
    return v.kern.random_actions(v, key, out)


def random_actions(batch, key: RngKey) -> np.ndarray:
    """Host-array version with the reference's return type (agents.py:33-46).

    Always a fresh array: when the fused sampler wrote into a caller's pinned host buffer, the
    launching stream is synchronised first (the kernel writes it asynchronously) and the buffer
    is copied, so the result neither races the kernel nor aliases a buffer the caller reuses."""
    a = random_actions_device(batch, key)
    if a.device.type == "cpu":
        import torch

        torch.cuda.current_stream(batch._v.device).synchronize()
        return a.numpy().copy()
    return a.cpu().numpy()


class RolloutResult:
    """First-episode outcome of every slot of a batched random rollout."""

    __slots__ = ("game_id", "returns", "lengths", "steps")

    def __init__(self, game_id, returns, lengths, steps):
        self.game_id = game_id
        self.returns = returns      # float32 [n, players], rewards by player at the episode's end
        self.lengths = lengths      # int32 [n], steps of the episode (step_count when it ended)
        self.steps = steps          # batch steps taken until every slot had finished once


def rollout(game, n: int, seed: int, *, max_steps: int | None = None, check_every: int = 16) -> RolloutResult:
    """Uniform-random rollouts to the end of the episode for n slots (agents.py:113-116, batched).

    Every slot plays the reference's random policy on the BatchSession key schedule
    (bench.py:54-83) -- the same trajectories as the reference's own ``BatchSession`` +
    ``random_actions`` loop -- until its first episode ends. The step kernel samples the next
    actions itself, ``bbk_latch_finished`` records each slot's first outcome on the device, and the
    host only polls a finished-slot counter every ``check_every`` steps.
    """
    import torch

    from . import _native as nat
    from .session import BatchSession

    sess = BatchSession(game, n, seed, max_steps=max_steps, validate=False)
    v0 = sess.batch._v
    dev = v0.device
    players = sess.gdef.spec.num_players
    done = torch.zeros(n, dtype=torch.uint8, device=dev)
    ret = torch.zeros((n, players), dtype=torch.float32, device=dev)
    length = torch.zeros(n, dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = nat.stream_handle(dev)
    t = 0
    while True:
        b = sess.step(sess.sample_random_actions())
        d = b.device
        nat.check(nat.lib().bbk_latch_finished(nat.ptr(d.terminated), nat.ptr(d.truncated), nat.ptr(d.rewards),
                                               nat.ptr(d.step_count), players, n, nat.ptr(done), nat.ptr(ret),
                                               nat.ptr(length), nat.ptr(count), stream), "bbk_latch_finished")
        t += 1
        if t % check_every == 0 or t >= (max_steps or sess.gdef.max_steps) + 1:
            if int(count.item()) >= n:
                break
    return RolloutResult(sess.gdef.game_id, ret.cpu().numpy(), length.cpu().numpy(), t)


# ----------------------------------------------------------------- search agents and matches
from .search import mcts_actions, mcts_agent  # noqa: E402  (batched UCT search, agents.py:63-123)


@dataclass(frozen=True)
class MatchResult:
    """Aggregate outcome of one pairing (reference elo.py:22-35)."""

    game_id: str
    agent_a: str
    agent_b: str
    wins_a: int
    wins_b: int
    draws: int

    @property
    def total(self) -> int:
        return self.wins_a + self.wins_b + self.draws


@dataclass(frozen=True)
class AgentPolicy:
    """A named decision function (agents.py:134-144). ``simulations`` marks the UCT agent, which
    the batched match runner searches on the device for all its games at once."""

    name: str
    fn: Callable
    requires_perfect_information: bool = False
    simulations: int = 0

    def __call__(self, state: EnvState, key: RngKey) -> int:
        return self.fn(state, key)


def random_policy() -> AgentPolicy:
    return AgentPolicy("random", random_agent)


def mcts_policy(simulations: int = 32) -> AgentPolicy:
    def fn(state, key):
        return mcts_agent(state, key, simulations)

    return AgentPolicy(f"mcts{simulations}", fn, requires_perfect_information=True, simulations=simulations)


def _keys_at(states: np.ndarray, index: int) -> np.ndarray:
    from .rng import child_states_at

    return child_states_at(states, index)


def _random_choice(mask: np.ndarray, key_states: np.ndarray) -> np.ndarray:
    """random_agent per row: legal[key.randint(len(legal))] (agents.py:25-30); 0 for empty rows."""
    cnt = mask.sum(axis=1).astype(np.uint64)
    d = key_states.astype(np.uint64) % np.maximum(cnt, 1)
    cum = np.cumsum(mask, axis=1, dtype=np.int64)
    act = (cum <= d[:, None].astype(np.int64)).sum(axis=1)
    act[cnt == 0] = 0
    return act.astype(np.int64)


def play_games(game, players: tuple, keys) -> tuple:
    """``play_game(gdef, players, key)`` (agents.py:163-172) for every key at once, one slot per
    game: (rewards [G, 2], step_count [G]) of each game's final state. Games advance in lockstep; UCT moves of all
    games whose player to move is the same search agent are one batched device search."""
    from .core import resolve
    from .rng import key_state

    gdef = resolve(game)
    kern = gdef.batch_kernel
    g = len(keys)
    ks = np.asarray([key_state(k) for k in keys], dtype=np.uint64)
    limit = gdef.max_steps
    v = kern.init(gdef, None, g, limit, slot_keys=_keys_at(ks, 0).tolist())
    done = np.zeros(g, dtype=bool)
    final = np.zeros((g, gdef.spec.num_players), dtype=np.float32)
    length = np.zeros(g, dtype=np.int32)
    t = 0
    pools = {}
    while True:
        fin = np.asarray(v.terminated, dtype=bool) | np.asarray(v.truncated, dtype=bool)
        fresh = fin & ~done
        if fresh.any():
            final[fresh] = np.asarray(v.rewards)[fresh]
            length[fresh] = np.asarray(v.step_count)[fresh]
            done |= fresh
        if done.all():
            return final, length
        t += 1
        akeys = _keys_at(ks, 2 * t - 1)
        mask = np.asarray(v.legal_action_mask, dtype=bool)
        acts = _random_choice(mask, akeys)          # random agents, and the games already over
        cur = np.asarray(v.current_player)
        for p, agent in enumerate(players):
            if agent.simulations <= 0:
                if agent.fn is not random_agent:
                    raise ValueError(f"agent {agent.name!r} has no batched device form")
                continue
            rows = np.flatnonzero(~done & ~fin & (cur == p))
            if rows.size:
                acts[rows] = mcts_search_rows(v, rows, akeys[rows], agent.simulations, pools, p)
        v = kern.step(gdef, v, acts, None, limit, validate=True, slot_keys=_keys_at(ks, 2 * t).tolist())


def mcts_search_rows(v, rows, key_states, simulations, pools, tag):
    from . import search

    pool = pools.get((tag, len(rows)))
    if pool is None or not pool.fits(v.kern, v, len(rows), simulations):
        pool = search.SearchPool(v.kern, v, len(rows), simulations)
        pools[(tag, len(rows))] = pool
    return search.search(v, rows.tolist(), [int(k) for k in key_states], simulations, pool=pool).cpu().numpy()


def run_matches(game, agents: list, games_per_pair: int, key: RngKey) -> list:
    """Round-robin pairwise matches (agents.py:175-216) with every pairing's games played in
    parallel on the device; identical results to the reference's sequential runner."""
    from .core import UnsupportedGame, resolve

    gdef = resolve(game)
    if len(agents) < 2:
        raise ValueError("run_matches needs at least two agents")
    chance_or_hidden = gdef.chance_in_step or not gdef.perfect_information
    for agent in agents:
        if agent.requires_perfect_information and (chance_or_hidden or gdef.spec.num_players != 2):
            raise UnsupportedGame(f"{agent.name} does not support {gdef.game_id}")
    if gdef.spec.num_players != 2:
        raise UnsupportedGame(f"run_matches supports 2-player games, not {gdef.game_id}")
    if games_per_pair == 0:
        return []
    results = []
    pair_index = 0
    for i in range(len(agents)):
        for j in range(i + 1, len(agents)):
            pair_key = key.child(pair_index)
            pair_index += 1
            final, _ = play_games(gdef, (agents[i], agents[j]), [pair_key.child(g) for g in range(games_per_pair)])
            r0 = final[:, 0]
            results.append(MatchResult(gdef.game_id, agents[i].name, agents[j].name, int((r0 > 0).sum()),
                                       int((r0 < 0).sum()), int((r0 == 0).sum())))
    return results
